# round 2: fill with two rows per group (HELIOS_SAMPLE_FILL_PAIR) + unrolled relabel: parity, C2 split / bench.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HELIOS_SAMPLE_FILL_PAIR=1 timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py -x -q -k "not c3_full" > $out/pt_z.log 2>&1; echo "rc=$?" >> $out/pt_z.log; tail -2 $out/pt_z.log
timeout 900 python -m pytest tests/test_gpu_sample.py -x -q > $out/pt_z0.log 2>&1; echo "rc=$?" >> $out/pt_z0.log; tail -2 $out/pt_z0.log
for p in 1 2; do
HELIOS_SAMPLE_FILL_PAIR=1 timeout 600 python tools/exp_split.py C2 > $out/split_z_pair_p$p.json 2>/dev/null; cat $out/split_z_pair_p$p.json
timeout 600 python tools/exp_split.py C2 > $out/split_z_base_p$p.json 2>/dev/null; cat $out/split_z_base_p$p.json
HELIOS_SAMPLE_FILL_PAIR=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bz_c2_pair_p$p.json 2>$out/bz_c2_pair.err; tail -c 60 $out/bz_c2_pair_p$p.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bz_c2_base_p$p.json 2>$out/bz_c2_base.err; tail -c 60 $out/bz_c2_base_p$p.json
done
HELIOS_SAMPLE_FILL_PAIR=1 timeout 900 python bench.py --no-cpu-baseline > $out/bz_c3_pair.json 2>$out/bz_c3_pair.err; tail -c 60 $out/bz_c3_pair.json
