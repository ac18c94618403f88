run() { n=$1; shift; timeout 1500 env "$@" > gpurun_out/b22_$n.json 2> gpurun_out/b22_$n.err; }
run c4 python bench.py --config C4 --steps 40 --warmup 3 --no-cpu-baseline
run c1 python bench.py --config C1 --steps 1000
