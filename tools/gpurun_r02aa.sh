# round 2: K4 with 4 loads in flight per lane (80 registers instead of 113) in the pipeline, same box A/B.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HELIOS_GATHER_VU=4 timeout 600 python -m pytest tests/test_gpu_gather.py -x -q -k "three_tiers or row_sizes" > $out/pt_aa.log 2>&1; echo "rc=$?" >> $out/pt_aa.log; tail -2 $out/pt_aa.log
for p in 1 2; do
  HELIOS_GATHER_VU=4 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baa_c2_vu4_p$p.json 2>/dev/null; tail -c 60 $out/baa_c2_vu4_p$p.json
  timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baa_c2_vu8_p$p.json 2>/dev/null; tail -c 60 $out/baa_c2_vu8_p$p.json
done
HELIOS_GATHER_VU=4 HELIOS_GATHER_CTAS_PER_SM=2 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baa_c2_vu4_2cta.json 2>/dev/null; tail -c 60 $out/baa_c2_vu4_2cta.json
HELIOS_GATHER_VU=4 timeout 600 python tools/exp_k4.py C2 20 > $out/k4aa.jsonl 2>/dev/null; cat $out/k4aa.jsonl
HELIOS_GATHER_VU=4 timeout 900 python bench.py --no-cpu-baseline > $out/baa_c3_vu4.json 2>/dev/null; tail -c 60 $out/baa_c3_vu4.json
timeout 900 python bench.py --no-cpu-baseline > $out/baa_c3_vu8.json 2>/dev/null; tail -c 60 $out/baa_c3_vu8.json
