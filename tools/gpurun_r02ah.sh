# round 2: windowed resolve in the fused HBM-only gather (HELIOS_GATHER_WINDOW): parity, K4 alone on C2's
# lists, C2 A/B on one box.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_gather.py tests/test_gpu_fullsize.py -x -q -k "direct or c2" > $out/pt_ah.log 2>&1; echo "rc=$?" >> $out/pt_ah.log; tail -3 $out/pt_ah.log
for v in "0 1 4" "1 1 4" "0 2 4" "1 2 4" "1 1 8" "1 2 8" "1 3 4"; do set -- $v
  HELIOS_GATHER_WINDOW=$1 HELIOS_GATHER_CTAS_PER_SM=$2 HELIOS_GATHER_VU=$3 timeout 600 python tools/exp_k4.py C2 20 2>/dev/null | sed "s/^/{\"window\": $1, \"per_sm\": $2, \"vu\": $3, \"r\": /; s/$/}/" >> $out/k4ah.jsonl
done
cat $out/k4ah.jsonl
for p in 1 2; do
  for v in "0 1 4" "1 1 4" "1 1 8" "1 2 4"; do set -- $v
    HELIOS_GATHER_WINDOW=$1 HELIOS_GATHER_CTAS_PER_SM=$2 HELIOS_GATHER_VU=$3 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bah_c2_w$1_s$2_v$3_p$p.json 2>/dev/null; tail -c 60 $out/bah_c2_w$1_s$2_v$3_p$p.json
  done
done
