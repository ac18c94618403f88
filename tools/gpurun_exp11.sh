run() { n=$1; shift; timeout 300 env "$@" > gpurun_out/b11_$n.json 2> gpurun_out/b11_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
run k1h2 HELIOS_GATHER_CTAS_PER_SM=1 HELIOS_HOST_WARPS_PER_8=2 $B
run k1h4 HELIOS_GATHER_CTAS_PER_SM=1 HELIOS_HOST_WARPS_PER_8=4 $B
run k2h2 HELIOS_GATHER_CTAS_PER_SM=2 HELIOS_HOST_WARPS_PER_8=2 $B
run k1h1d12 HELIOS_GATHER_CTAS_PER_SM=1 $B --depth 12
run k1h1 HELIOS_GATHER_CTAS_PER_SM=1 $B
