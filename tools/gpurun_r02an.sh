# round 2: evict-first L2 policy on the fill's CSR index reads (HELIOS_SAMPLE_IDX_EVICT) and on K4's
# HBM-row copies (HELIOS_GATHER_EVICT_LISTS): C2 / C3 A/B on one box (the bench checks parity).
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_plan.py -x -q > $out/pt_an.log 2>&1; echo "rc=$?" >> $out/pt_an.log; tail -3 $out/pt_an.log
for p in 1 2; do
for v in 0 1; do
  HELIOS_SAMPLE_IDX_EVICT=$v timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/ban_c2_i${v}_p$p.json 2>/dev/null; tail -c 60 $out/ban_c2_i${v}_p$p.json
done
done
for p in 1 2; do
for v in "0 0" "0 1" "1 0" "1 1"; do set -- $v
  HELIOS_SAMPLE_IDX_EVICT=$1 HELIOS_GATHER_EVICT_LISTS=$2 timeout 900 python bench.py --no-cpu-baseline --steps 1500 > $out/ban_c3_i$1_l$2_p$p.json 2>/dev/null; tail -c 60 $out/ban_c3_i$1_l$2_p$p.json
done
done
