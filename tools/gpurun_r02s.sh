# round 2: C3 split host kernel vs combined at depth 12 / 16 / 24 (two passes, same box) and the C1/C4 CQ backoff.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
for pass in 1 2; do
for d in 12 16 24; do
  timeout 900 python bench.py --no-cpu-baseline --depth $d > $out/bs_c3_d${d}_p$pass.json 2>$out/bs_c3_d${d}_p$pass.err; tail -c 60 $out/bs_c3_d${d}_p$pass.json
  HELIOS_GATHER_SPLIT_HOST=1 timeout 900 python bench.py --no-cpu-baseline --depth $d > $out/bs_c3_split_d${d}_p$pass.json 2>$out/bs_c3_split_d${d}_p$pass.err; tail -c 60 $out/bs_c3_split_d${d}_p$pass.json
done; done
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 > $out/bs_c1.json 2>$out/bs_c1.err
timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 40 > $out/bs_c4.json 2>$out/bs_c4.err
