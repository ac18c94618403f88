# round 2: plan groups (parity + C2/C3 benches) and the green-context IO partition (NEXT-3).
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_gather.py tests/test_gpu_sample.py -x -q > $out/pt_m.log 2>&1; echo "rc=$?" >> $out/pt_m.log; tail -3 $out/pt_m.log
for gd in "1 12" "2 6" "4 3" "4 4" "3 4"; do set -- $gd; timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --group $1 --depth $2 > $out/bm_c2_g$1d$2.json 2>$out/bm_c2_g$1d$2.err; tail -c 100 $out/bm_c2_g$1d$2.json; done
for gd in "2 6" "4 3"; do set -- $gd; timeout 900 python bench.py --no-cpu-baseline --group $1 --depth $2 > $out/bm_c3_g$1d$2.json 2>$out/bm_c3_g$1d$2.err; tail -c 100 $out/bm_c3_g$1d$2.json; done
for m in 8 16 48; do timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 --io-sms $m > $out/bm_c1_sm$m.json 2>$out/bm_c1_sm$m.err; tail -c 100 $out/bm_c1_sm$m.json; done
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 > $out/bm_c1_sm0.json 2>$out/bm_c1_sm0.err
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2" > $out/pt_m_full.log 2>&1; echo "rc=$?" >> $out/pt_m_full.log; tail -3 $out/pt_m_full.log
