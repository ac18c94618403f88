# round 2: home region shrinks one halving per batch at most: sampler / gather / plan / full-size parity, C2 / C3.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py tests/test_gpu_gather.py tests/test_gpu_multirank.py -x -q --durations=5 > $out/pt_ay.log 2>&1; echo "rc=$?" >> $out/pt_ay.log; tail -9 $out/pt_ay.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ay.log 2>&1; echo "rc=$?" >> $out/smoke_ay.log; tail -2 $out/smoke_ay.log
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bay_c2.json 2>/dev/null; tail -c 60 $out/bay_c2.json
timeout 900 python bench.py > $out/bay_c3.json 2>/dev/null; tail -c 60 $out/bay_c3.json
