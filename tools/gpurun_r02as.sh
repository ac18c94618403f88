# round 2: confirm the fill grid (HELIOS_FILL_CTAS_PER_SM) and C2 plan depth under the new L2 policies, and
# the C3 stager reservation, two passes on one box.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for p in 1 2; do
for v in "2 12" "3 12" "3 16" "4 12" "4 16"; do set -- $v
  HELIOS_FILL_CTAS_PER_SM=$1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --depth $2 > $out/bas_c2_f$1_d$2_p$p.json 2>/dev/null; tail -c 60 $out/bas_c2_f$1_d$2_p$p.json
done
for v in "2 0.7" "3 0.7" "3 0.6"; do set -- $v
  HELIOS_FILL_CTAS_PER_SM=$1 timeout 900 python bench.py --no-cpu-baseline --steps 1500 --stage-reserve $2 > $out/bas_c3_f$1_r$2_p$p.json 2>/dev/null; tail -c 60 $out/bas_c3_f$1_r$2_p$p.json
done
done
