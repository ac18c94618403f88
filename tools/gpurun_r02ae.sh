# round 2: segment-packed fill as the default: sampler / plan / full-size parity (both fill variants), C2 + C3 default.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_sample.py tests/test_gpu_plan.py tests/test_gpu_fullsize.py -x -q > $out/pt_ae.log 2>&1; echo "rc=$?" >> $out/pt_ae.log; tail -2 $out/pt_ae.log
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bae_c2.json 2>/dev/null; tail -c 60 $out/bae_c2.json
timeout 900 python bench.py --no-cpu-baseline > $out/bae_c3.json 2>/dev/null; tail -c 60 $out/bae_c3.json
