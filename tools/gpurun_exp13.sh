timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest13.log 2>&1; echo "rc=$?" >> gpurun_out/pytest13.log; tail -2 gpurun_out/pytest13.log
run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b13_$n.json 2> gpurun_out/b13_$n.err; }
run c3 python bench.py
run c2 python bench.py --config C2 --no-cpu-baseline
run c3st python bench.py --no-cpu-baseline --host-staged 0.6
