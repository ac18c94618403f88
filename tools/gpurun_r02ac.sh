# round 2 validation of the final defaults (K4 VU=4, fill <= 2 CTAs/SM, split host kernel, 24 slots with a
# host tier, PDL off for host-tier plans): full GPU suite, smoke, default bench (C3) + C2, ncu launch list.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $out/build_ac.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pt_ac.log 2>&1; echo "rc=$?" >> $out/pt_ac.log; tail -3 $out/pt_ac.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ac.log 2>&1; echo "rc=$?" >> $out/smoke_ac.log; tail -2 $out/smoke_ac.log
timeout 900 python bench.py > $out/bac_c3.json 2>$out/bac_c3.err; tail -c 200 $out/bac_c3.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bac_c2.json 2>$out/bac_c2.err; tail -c 100 $out/bac_c2.json
timeout 600 python tools/exp_split.py C2 > $out/split_ac.json 2>/dev/null; cat $out/split_ac.json
timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 40 > $out/bac_c4.json 2>$out/bac_c4.err; tail -c 100 $out/bac_c4.json
timeout 600 python bench.py --config C1 --no-cpu-baseline --steps 1000 > $out/bac_c1.json 2>$out/bac_c1.err; tail -c 100 $out/bac_c1.json
timeout 1200 bash tools/profile_c3.sh r02ac_c3 "k_gather_lists|k_gather_host|k_lookup" > /dev/null 2>&1
timeout 900 bash tools/profile_c3.sh r02ac_c2 "k_gather_lists|k_lookup|k_fill_insert" --config C2 > /dev/null 2>&1
ls $out | grep ac
