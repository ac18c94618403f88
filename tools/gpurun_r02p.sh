# round 2: shared-memory tile dedup (HELIOS_SAMPLE_DEDUP=smem): parity, then C2 split / benches and C3.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sample.py -x -q > $out/pt_p.log 2>&1; echo "rc=$?" >> $out/pt_p.log; tail -3 $out/pt_p.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k c2 > $out/pt_p_full.log 2>&1; echo "rc=$?" >> $out/pt_p_full.log; tail -3 $out/pt_p_full.log
HELIOS_SAMPLE_DEDUP=smem timeout 600 python tools/exp_split.py C2 > $out/split_p_smem.json 2>$out/split_p_smem.err; cat $out/split_p_smem.json
timeout 600 python tools/exp_split.py C2 > $out/split_p_global.json 2>$out/split_p_global.err; cat $out/split_p_global.json
HELIOS_SAMPLE_DEDUP=smem timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bp_c2_smem.json 2>$out/bp_c2_smem.err; tail -c 100 $out/bp_c2_smem.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bp_c2_global.json 2>$out/bp_c2_global.err; tail -c 100 $out/bp_c2_global.json
HELIOS_SAMPLE_DEDUP=smem timeout 900 python bench.py --no-cpu-baseline > $out/bp_c3_smem.json 2>$out/bp_c3_smem.err; tail -c 100 $out/bp_c3_smem.json
