set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for f in 0.5 0.6 0.75 1.0; do timeout 900 python bench.py --no-cpu-baseline --host-staged $f > $out/bf_c3_f$f.json 2>$out/bf_c3_f$f.err; tail -c 150 $out/bf_c3_f$f.json; done
timeout 900 python bench.py --no-cpu-baseline --host-staged 0.6 --stage-workers 14 > $out/bf_c3_f0.6w14.json 2>$out/bf_c3_f0.6w14.err
