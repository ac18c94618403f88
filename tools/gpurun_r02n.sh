# round 2: plan groups benches (C2/C3), replicated HBM tier (2 ranks on 1 GPU), C1 IO variants.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_multirank.py -x -q > $out/pt_n.log 2>&1; echo "rc=$?" >> $out/pt_n.log; tail -3 $out/pt_n.log
for gd in "2 6" "4 3" "4 4" "3 4" "4 6"; do set -- $gd; timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --group $1 --depth $2 > $out/bn_c2_g$1d$2.json 2>$out/bn_c2_g$1d$2.err; tail -c 100 $out/bn_c2_g$1d$2.json; done
for gd in "2 6" "4 3"; do set -- $gd; timeout 900 python bench.py --no-cpu-baseline --group $1 --depth $2 > $out/bn_c3_g$1d$2.json 2>$out/bn_c3_g$1d$2.err; tail -c 100 $out/bn_c3_g$1d$2.json; done
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 --io-sync > $out/bn_c1_sync.json 2>$out/bn_c1_sync.err
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 --io-ctas 4 > $out/bn_c1_ctas4.json 2>$out/bn_c1_ctas4.err
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 --depth 2 > $out/bn_c1_d2.json 2>$out/bn_c1_d2.err
