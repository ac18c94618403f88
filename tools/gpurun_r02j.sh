# round 2: stager reservation sweep on C3, fixed link probe, C2 gather grid in the whole pipeline.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_plan.py -x -q > $out/pt_j.log 2>&1; echo "rc=$?" >> $out/pt_j.log; tail -2 $out/pt_j.log
for r in 0.6 0.4 0.8 0; do timeout 900 python bench.py --no-cpu-baseline --stage-reserve $r > $out/bj_c3_r$r.json 2>$out/bj_c3_r$r.err; tail -c 120 $out/bj_c3_r$r.json; done
for v in 1 2; do HELIOS_GATHER_CTAS_PER_SM=$v timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bj_c2_g$v.json 2>$out/bj_c2_g$v.err; done
