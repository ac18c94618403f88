# round 2: green-context IO partition (NEXT-3) parity + sweeps on C1/C4; C4 host tier on/off (NEXT-4).
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -k "green or io_ring or three_tiers" > $out/pt_l.log 2>&1; echo "rc=$?" >> $out/pt_l.log; tail -3 $out/pt_l.log
for m in 0 8 16 24 48; do timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 --io-sms $m > $out/bl_c1_sm$m.json 2>$out/bl_c1_sm$m.err; tail -c 100 $out/bl_c1_sm$m.json; done
for m in 0 16 48; do timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 40 --io-sms $m > $out/bl_c4_sm$m.json 2>$out/bl_c4_sm$m.err; tail -c 100 $out/bl_c4_sm$m.json; done
timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 40 --host-frac 0 > $out/bl_c4_nohost.json 2>$out/bl_c4_nohost.err; tail -c 100 $out/bl_c4_nohost.json
