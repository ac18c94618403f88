# round 2: yielding readback wait (e2e with stagers), reference arm smoke, C3 default twice.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_plan.py -x -q > $out/pt_v.log 2>&1; echo "rc=$?" >> $out/pt_v.log; tail -2 $out/pt_v.log
for p in 1 2; do timeout 900 python bench.py --no-cpu-baseline > $out/bv_c3_p$p.json 2>$out/bv_c3_p$p.err; tail -c 60 $out/bv_c3_p$p.json; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/bv_ref.json 2>$out/bv_ref.err; tail -c 400 $out/bv_ref.json
