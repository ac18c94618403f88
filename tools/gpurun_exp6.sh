run() { n=$1; shift; timeout 300 env "$@" > gpurun_out/b6_$n.json 2> gpurun_out/b6_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1 --steps 3000"
run c2d6 $B --config C2
run c2d8 $B --config C2 --depth 8
run c2d12 $B --config C2 --depth 12
run c2d16 $B --config C2 --depth 16
run c2d6nopdl HELIOS_NO_PDL=1 $B --config C2
run c2d12nopdl HELIOS_NO_PDL=1 $B --config C2 --depth 12
run c3d12 $B --depth 12
run c3d6nopdl HELIOS_NO_PDL=1 $B
