set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for w in 8 14; do timeout 900 python bench.py --no-cpu-baseline --stage-workers $w > $out/be_c3_w$w.json 2>$out/be_c3_w$w.err; tail -c 200 $out/be_c3_w$w.json; done
timeout 900 python bench.py --no-cpu-baseline --zero-copy > $out/be_c3_zc.json 2>$out/be_c3_zc.err; tail -c 200 $out/be_c3_zc.json
