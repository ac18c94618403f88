# round 2: count-scan / assign tile size A/B builds (HELIOS_SCAN_ITEMS = 2 / 8 vs the default 4) on C2 and C3,
# C3 stager reservation / fill grid, and C2 sampling-only at the bench depth; one box, two passes.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
HELIOS_LIB=si2 timeout 900 python -m pytest tests/test_gpu_sample.py -x -q -k "chain or c1_full or home" > $out/pt_aw2.log 2>&1; echo "rc=$?" >> $out/pt_aw2.log; tail -2 $out/pt_aw2.log
HELIOS_LIB=si8 timeout 900 python -m pytest tests/test_gpu_sample.py -x -q -k "chain or c1_full or home" > $out/pt_aw8.log 2>&1; echo "rc=$?" >> $out/pt_aw8.log; tail -2 $out/pt_aw8.log
for p in 1 2; do
for v in def si2 si8; do
  L=""; [ $v != def ] && L=$v
  env ${L:+HELIOS_LIB=$L} timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baw_c2_${v}_p$p.json 2>/dev/null; tail -c 60 $out/baw_c2_${v}_p$p.json
done
done
for p in 1 2; do
for v in "def 4 0.7" "si2 4 0.7" "def 6 0.7" "def 4 0.6"; do set -- $v
  L=""; [ $1 != def ] && L=$1
  env ${L:+HELIOS_LIB=$L} HELIOS_FILL_CTAS_PER_SM=$2 timeout 900 python bench.py --no-cpu-baseline --steps 1500 --stage-reserve $3 > $out/baw_c3_$1_f$2_r$3_p$p.json 2>/dev/null; tail -c 60 $out/baw_c3_$1_f$2_r$3_p$p.json
done
done
