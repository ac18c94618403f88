# round 2: fill grid x plan depth sweep under the new L2 policies (C2 two passes, C3 one).
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for p in 1 2; do
for v in "4 16" "6 16" "8 16" "4 20" "6 20" "6 24"; do set -- $v
  HELIOS_FILL_CTAS_PER_SM=$1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --depth $2 > $out/bat_c2_f$1_d$2_p$p.json 2>/dev/null; tail -c 60 $out/bat_c2_f$1_d$2_p$p.json
done
done
for v in "3 24" "4 24" "6 24" "4 32"; do set -- $v
  HELIOS_FILL_CTAS_PER_SM=$1 timeout 900 python bench.py --no-cpu-baseline --steps 1500 --depth $2 > $out/bat_c3_f$1_d$2.json 2>/dev/null; tail -c 60 $out/bat_c3_f$1_d$2.json
done
