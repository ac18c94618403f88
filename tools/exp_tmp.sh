run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b21_$n.json 2> gpurun_out/b21_$n.err; }
run c2 python bench.py --config C2 --no-cpu-baseline
run c3 python bench.py
