# round 2: host-tier rows in their own small kernel (HELIOS_GATHER_SPLIT_HOST): parity + C3 / C1 benches.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -k "split_host or three_tiers" > $out/pt_r.log 2>&1; echo "rc=$?" >> $out/pt_r.log; tail -3 $out/pt_r.log
HELIOS_GATHER_SPLIT_HOST=1 timeout 900 python bench.py --no-cpu-baseline > $out/br_c3_split.json 2>$out/br_c3_split.err; tail -c 100 $out/br_c3_split.json
HELIOS_GATHER_SPLIT_HOST=1 timeout 900 python bench.py --no-cpu-baseline --depth 16 > $out/br_c3_split_d16.json 2>$out/br_c3_split_d16.err; tail -c 100 $out/br_c3_split_d16.json
HELIOS_GATHER_SPLIT_HOST=1 timeout 900 python bench.py --no-cpu-baseline --zero-copy > $out/br_c3_split_zc.json 2>$out/br_c3_split_zc.err; tail -c 100 $out/br_c3_split_zc.json
timeout 900 python bench.py --no-cpu-baseline > $out/br_c3.json 2>$out/br_c3.err; tail -c 100 $out/br_c3.json
HELIOS_GATHER_SPLIT_HOST=1 timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 > $out/br_c1_split.json 2>$out/br_c1_split.err; tail -c 100 $out/br_c1_split.json
