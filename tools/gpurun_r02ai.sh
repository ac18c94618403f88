# round 2: candidate-marking inserts (HELIOS_SAMPLE_CAND): sampler parity in every mode, C2 full size,
# sampling-only and whole-step A/B on C2, C3 A/B.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py -x -q -k "not c3_full" > $out/pt_ai.log 2>&1; echo "rc=$?" >> $out/pt_ai.log; tail -3 $out/pt_ai.log
for p in 1 2; do
  for v in 1 0; do
    HELIOS_SAMPLE_CAND=$v timeout 600 python tools/exp_split.py C2 > $out/split_ai_c$v_p$p.json 2>/dev/null; echo "{\"cand\": $v, \"split\": $(cat $out/split_ai_c$v_p$p.json)}" >> $out/split_ai.jsonl
    HELIOS_SAMPLE_CAND=$v timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bai_c2_c${v}_p$p.json 2>/dev/null; tail -c 60 $out/bai_c2_c${v}_p$p.json
  done
done
cat $out/split_ai.jsonl
for v in 1 0; do
  HELIOS_SAMPLE_CAND=$v timeout 900 python bench.py --no-cpu-baseline > $out/bai_c3_c${v}.json 2>/dev/null; tail -c 60 $out/bai_c3_c${v}.json
done
