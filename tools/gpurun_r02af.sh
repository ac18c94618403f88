# round 2: fused lookup+gather for HBM-only caches (HELIOS_GATHER_DIRECT): parity (single + 2 ranks, C2 full
# size), C2 A/B on one box, K4-only isolation.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_gather.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -x -q -k "direct or multirank or two_ranks or c2" > $out/pt_af.log 2>&1; echo "rc=$?" >> $out/pt_af.log; tail -2 $out/pt_af.log
for p in 1 2; do
  timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baf_c2_direct_p$p.json 2>/dev/null; tail -c 60 $out/baf_c2_direct_p$p.json
  HELIOS_GATHER_DIRECT=0 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baf_c2_k3k4_p$p.json 2>/dev/null; tail -c 60 $out/baf_c2_k3k4_p$p.json
done
timeout 600 python tools/exp_split.py C2 > $out/split_af.json 2>/dev/null; cat $out/split_af.json
timeout 600 python tools/exp_k4.py C2 20 > $out/k4af.jsonl 2>/dev/null; cat $out/k4af.jsonl
