export CUDA_MODULE_LOADING=EAGER
timeout 300 python tools/host_slots.py /tmp/c3s 48 > gpurun_out/host_slots2.json 2>/dev/null
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/hostorder tools/hostorder.cu
for nz in 148 592; do timeout 240 /tmp/hostorder /tmp/c3s 99900000 512 $nz > gpurun_out/hostorder_noise$nz.jsonl 2>&1; done
for a in "--depth 1" "--depth 1 --shared-link" "--depth 3"; do
  n=$(echo "c3$a" | tr -d ' .-')
  timeout 400 python bench.py --no-cpu-baseline --steps 1000 --parity-batches 1 $a > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
done
