# round 2: home-region floor (1/8 of the worst-case table): sampler + full-size C2 + plan parity, C2 / C3 bench.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py tests/test_gpu_gather.py -x -q --durations=8 -k "not c3_full" > $out/pt_ax.log 2>&1; echo "rc=$?" >> $out/pt_ax.log; tail -14 $out/pt_ax.log
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bax_c2.json 2>/dev/null; tail -c 60 $out/bax_c2.json
timeout 900 python bench.py --no-cpu-baseline --steps 1500 > $out/bax_c3.json 2>/dev/null; tail -c 60 $out/bax_c3.json
