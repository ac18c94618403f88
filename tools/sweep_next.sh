#!/bin/bash
# SURVEY §8(f) NEXT-rows experiments (one JSON line per run into gpurun_out/next_r01.jsonl).
out=${GRAFT_REPO_ROOT:-.}/gpurun_out/next_r01.jsonl
: > $out
run() { tag=$1; shift; r=$(timeout 900 python bench.py --no-cpu-baseline --parity-batches 1 "$@" 2>/dev/null | tail -1); echo "{\"tag\": \"$tag\", \"args\": \"$*\", \"result\": ${r:-null}}" >> $out; }
# NEXT-3: IO stack, decoupled vs GIDS-style coupled, CTA budget sweep (C1: file tier 50%)
for m in async sync; do for ctas in 1 2 4 8 32 128; do
  if [ $m = sync ]; then run io_$m\_$ctas --config C1 --steps 400 --io-ctas $ctas --io-sync; else run io_$m\_$ctas --config C1 --steps 400 --io-ctas $ctas; fi
done; done
# NEXT-4: tier ablations on C3 (GPU cache on/off and size; host tier on/off -> file)
run tiers_c3_hbm0 --steps 500 --hbm-frac 0 --host-frac 1
run tiers_c3_hbm20 --steps 1000 --hbm-frac 0.2 --host-frac 0.8
run tiers_c3_hbm50 --steps 1000 --hbm-frac 0.5 --host-frac 0.5
run tiers_c3_hbm100 --steps 2000 --hbm-frac 1 --host-frac 0
# NEXT-2: host-resident topology (sampling over PCIe, UVA) vs HBM topology
run topo_host_c2 --config C2 --steps 300 --topo-host
run topo_host_c3 --steps 300 --topo-host
# NEXT-4 (C4 scaled): host tier on vs off, and the IO CTA budget on a disk-bound config
run c4_default --config C4 --steps 20 --warmup 3
run c4_nohost --config C4 --steps 10 --warmup 2 --host-frac 0
run c4_sync32 --config C4 --steps 20 --warmup 3 --io-sync
echo done
