run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/b4_$n.json 2> gpurun_out/b4_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
run l2 HELIOS_PLAN_LINKS=2 $B
run l3 HELIOS_PLAN_LINKS=3 $B
run l6 HELIOS_PLAN_LINKS=4 $B --depth 8
run st_shared HELIOS_PLAN_LINKS=1 $B --host-staged 0.6 --shared-link
run st_l2 HELIOS_PLAN_LINKS=2 $B --host-staged 0.6
