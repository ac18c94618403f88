timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_gather.py -x -q > gpurun_out/pytest5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest5.log; tail -2 gpurun_out/pytest5.log
run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b5_$n.json 2> gpurun_out/b5_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
run def $B
run st6 $B --host-staged 0.6
run st7w12 $B --host-staged 0.7 --stage-workers 12
run c2 $B --config C2
