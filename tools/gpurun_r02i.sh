# round 2 (re-entry): validate HEAD on a fresh box: full GPU suite, default bench (C3), C2, launch list.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pt_i.log 2>&1; echo "rc=$?" >> $out/pt_i.log; tail -3 $out/pt_i.log
timeout 900 python bench.py > $out/bi_c3.json 2>$out/bi_c3.err; tail -c 300 $out/bi_c3.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bi_c2.json 2>$out/bi_c2.err; tail -c 300 $out/bi_c2.json
timeout 600 python tools/exp_split.py C2 > $out/split_i_c2.json 2>$out/split_i_c2.err; cat $out/split_i_c2.json
