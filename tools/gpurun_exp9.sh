run() { n=$1; shift; timeout 300 env "$@" > gpurun_out/b9_$n.json 2> gpurun_out/b9_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 2"
run c2t256k HELIOS_TABLE_SLOTS=262144 $B --config C2
run c2t512k HELIOS_TABLE_SLOTS=524288 $B --config C2
run c3t256k HELIOS_TABLE_SLOTS=262144 $B
