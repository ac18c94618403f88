# round 2: two-level batch table (dense 2^18-slot primary + worst-case secondary), candidate inserts,
# evict-first fused gather: parity (every sampler mode incl. a 1,024-slot primary, C2 full size, plans),
# C2 / C3 A/B.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_sample.py tests/test_gpu_gather.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py -x -q -k "not c3_full" > $out/pt_ak.log 2>&1; echo "rc=$?" >> $out/pt_ak.log; tail -3 $out/pt_ak.log
for p in 1 2; do
for v in "262144 1 1" "262144 1 0" "0 1 1" "262144 0 1" "0 1 0"; do set -- $v
  HELIOS_TABLE_SLOTS=$1 HELIOS_SAMPLE_CAND=$2 HELIOS_GATHER_EVICT=$3 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bak_c2_t$1_c$2_e$3_p$p.json 2>/dev/null; tail -c 60 $out/bak_c2_t$1_c$2_e$3_p$p.json
done
done
for v in "262144 1" "0 1"; do set -- $v
  HELIOS_TABLE_SLOTS=$1 HELIOS_SAMPLE_CAND=$2 timeout 900 python bench.py --no-cpu-baseline > $out/bak_c3_t$1_c$2.json 2>/dev/null; tail -c 60 $out/bak_c3_t$1_c$2.json
done
