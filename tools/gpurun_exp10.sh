run() { n=$1; shift; timeout 300 env "$@" > gpurun_out/b10_$n.json 2> gpurun_out/b10_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
for k in 1 2; do
run c3k$k HELIOS_GATHER_CTAS_PER_SM=$k $B
run c3st6k$k HELIOS_GATHER_CTAS_PER_SM=$k $B --host-staged 0.6
run c2k$k HELIOS_GATHER_CTAS_PER_SM=$k $B --config C2
done
run c3st6k4 $B --host-staged 0.6
