timeout 900 python -m pytest tests/test_gpu_plan.py -x -q > gpurun_out/pytest14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest14.log; tail -2 gpurun_out/pytest14.log
run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b14_$n.json 2> gpurun_out/b14_$n.err; }
run c2 python bench.py --config C2 --no-cpu-baseline
run c3 python bench.py --no-cpu-baseline
