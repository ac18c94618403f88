run() { n=$1; shift; timeout 300 env "$@" > gpurun_out/b12_$n.json 2> gpurun_out/b12_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
run c3g74 HELIOS_GATHER_CTAS=74 $B
run c3g110 HELIOS_GATHER_CTAS=110 $B
run c3g222 HELIOS_GATHER_CTAS=222 $B
run c2g74 HELIOS_GATHER_CTAS=74 $B --config C2
run c2g148 HELIOS_GATHER_CTAS=148 $B --config C2
run c2g296 HELIOS_GATHER_CTAS=296 $B --config C2
