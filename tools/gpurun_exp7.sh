timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_gather.py -x -q > gpurun_out/pytest7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest7.log; tail -2 gpurun_out/pytest7.log
run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b7_$n.json 2> gpurun_out/b7_$n.err; }
run c3 python bench.py
run c2 python bench.py --config C2 --no-cpu-baseline
run c3d12 python bench.py --depth 12 --no-cpu-baseline
