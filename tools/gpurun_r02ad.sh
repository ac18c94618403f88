# round 2: segment-packed fill (HELIOS_FILL_SEG=1): parity, then C2 / C3 A/B on one box.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HELIOS_FILL_SEG=1 timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_plan.py tests/test_gpu_fullsize.py -x -q -k "not c3_full" > $out/pt_ad.log 2>&1; echo "rc=$?" >> $out/pt_ad.log; tail -2 $out/pt_ad.log
for p in 1 2; do
  HELIOS_FILL_SEG=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bad_c2_seg_p$p.json 2>/dev/null; tail -c 60 $out/bad_c2_seg_p$p.json
  timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bad_c2_base_p$p.json 2>/dev/null; tail -c 60 $out/bad_c2_base_p$p.json
done
HELIOS_FILL_SEG=1 timeout 600 python tools/exp_split.py C2 > $out/split_ad_seg.json 2>/dev/null; cat $out/split_ad_seg.json
HELIOS_FILL_SEG=1 HELIOS_FILL_CTAS_PER_SM=4 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bad_c2_seg_f4.json 2>/dev/null; tail -c 60 $out/bad_c2_seg_f4.json
HELIOS_FILL_SEG=1 timeout 900 python bench.py --no-cpu-baseline > $out/bad_c3_seg.json 2>/dev/null; tail -c 60 $out/bad_c3_seg.json
timeout 900 python bench.py --no-cpu-baseline > $out/bad_c3_base.json 2>/dev/null; tail -c 60 $out/bad_c3_base.json
