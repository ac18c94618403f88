# round 2: re-tune the C2 / C3 launch parameters under the new L2 policies (two passes each, one box):
# gather loads in flight / grid, fill CTAs per SM, plan depth; C3 depth and stager reservation.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for p in 1 2; do
for v in "4 1 2 12" "8 1 2 12" "4 2 2 12" "4 1 3 12" "4 1 2 16" "4 1 2 24"; do set -- $v
  HELIOS_GATHER_VU=$1 HELIOS_GATHER_CTAS_PER_SM=$2 HELIOS_FILL_CTAS_PER_SM=$3 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --depth $4 > $out/bar_c2_v$1_g$2_f$3_d$4_p$p.json 2>/dev/null; tail -c 60 $out/bar_c2_v$1_g$2_f$3_d$4_p$p.json
done
done
for v in "24 0.7" "32 0.7" "24 0.8" "24 0.6"; do set -- $v
  timeout 900 python bench.py --no-cpu-baseline --steps 1500 --depth $1 --stage-reserve $2 > $out/bar_c3_d$1_r$2.json 2>/dev/null; tail -c 60 $out/bar_c3_d$1_r$2.json
done
