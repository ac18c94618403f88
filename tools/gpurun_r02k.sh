# round 2: packed key|minpos table word (sampler parity + C2 split) and the batch-size (grouping) probe.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_plan.py -x -q > $out/pt_k.log 2>&1; echo "rc=$?" >> $out/pt_k.log; tail -2 $out/pt_k.log
timeout 600 python tools/exp_split.py C2 > $out/split_k_c2.json 2>$out/split_k_c2.err; cat $out/split_k_c2.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bk_c2.json 2>$out/bk_c2.err; tail -c 200 $out/bk_c2.json
timeout 900 python tools/exp_group.py > $out/group_k.json 2>$out/group_k.err; cat $out/group_k.json
timeout 900 python bench.py --no-cpu-baseline --stage-reserve 0.7 > $out/bk_c3_r0.7.json 2>$out/bk_c3_r0.7.err; tail -c 200 $out/bk_c3_r0.7.json
