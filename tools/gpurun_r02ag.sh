# round 2: fused HBM-only gather with loads staged through a cp.async shared-memory ring
# (HELIOS_GATHER_ASYNC=4/8): parity (C1 variants, C2 full size), K4 alone on C2's lists, C2 A/B.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_gather.py tests/test_gpu_fullsize.py -x -q -k "direct or c2" > $out/pt_ag.log 2>&1; echo "rc=$?" >> $out/pt_ag.log; tail -3 $out/pt_ag.log
for v in "0 1" "0 2" "4 1" "4 2" "4 3" "8 1"; do set -- $v
  HELIOS_GATHER_ASYNC=$1 HELIOS_GATHER_CTAS_PER_SM=$2 timeout 600 python tools/exp_k4.py C2 20 2>/dev/null | sed "s/^/{\"async\": $1, \"per_sm\": $2, \"r\": /; s/$/}/" >> $out/k4ag.jsonl
done
cat $out/k4ag.jsonl
for p in 1 2; do
  for v in "0 1" "4 1" "8 1" "4 2"; do set -- $v
    HELIOS_GATHER_ASYNC=$1 HELIOS_GATHER_CTAS_PER_SM=$2 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bag_c2_a$1_s$2_p$p.json 2>/dev/null; tail -c 60 $out/bag_c2_a$1_s$2_p$p.json
  done
done
