export CUDA_MODULE_LOADING=EAGER
timeout 300 python tools/host_slots.py /tmp/c3s 48 > /dev/null 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/hostnoise tools/hostnoise.cu
timeout 300 /tmp/hostnoise /tmp/c3s 99900000 512 148 > gpurun_out/hostnoise148.jsonl 2>&1

