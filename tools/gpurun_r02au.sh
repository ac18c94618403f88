# round 2: relabel / clear grid (HELIOS_TAIL_CTAS_PER_SM) at the new defaults, C2 two passes; sampling-only split.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for p in 1 2; do
for t in 2 4 8 1; do
  HELIOS_TAIL_CTAS_PER_SM=$t timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bau_c2_t${t}_p$p.json 2>/dev/null; tail -c 60 $out/bau_c2_t${t}_p$p.json
done
done
timeout 600 python tools/exp_split.py C2 > $out/split_au.json 2>/dev/null; cat $out/split_au.json
