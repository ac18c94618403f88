set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
grep -i AnonHugePages /proc/meminfo; cat /sys/kernel/mm/transparent_hugepage/enabled
for f in 0.6 1.0; do timeout 900 python bench.py --no-cpu-baseline --host-staged $f --stage-workers 14 > $out/bg_c3_f$f.json 2>$out/bg_c3_f$f.err; tail -c 150 $out/bg_c3_f$f.json; done
timeout 900 python bench.py --no-cpu-baseline --host-staged 1.0 --stage-workers 8 > $out/bg_c3_f1.0w8.json 2>$out/bg_c3_f1.0w8.err
