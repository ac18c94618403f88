# round 2: C3 reservation / stager sweep with the split host kernel at 24 slots (same box).
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
for r in 0.6 0.7 0.8 0.9; do timeout 900 python bench.py --no-cpu-baseline --stage-reserve $r > $out/bu_c3_r$r.json 2>$out/bu_c3_r$r.err; tail -c 60 $out/bu_c3_r$r.json; done
for w in 10 12; do timeout 900 python bench.py --no-cpu-baseline --stage-workers $w > $out/bu_c3_w$w.json 2>$out/bu_c3_w$w.err; tail -c 60 $out/bu_c3_w$w.json; done
timeout 900 python bench.py --no-cpu-baseline --depth 20 > $out/bu_c3_d20.json 2>$out/bu_c3_d20.err; tail -c 60 $out/bu_c3_d20.json
