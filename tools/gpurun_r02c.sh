# round 2: dynamic staged host tier (default), independent link probe, K4 flat w/ prefetch (HBM-only
# instantiation), C2 grid sweep, C3 default vs zero-copy.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gather.py tests/test_gpu_plan.py tests/test_gpu_fullsize.py tests/test_gpu_rng.py -x -q > $out/pt_c.log 2>&1; echo "rc=$?" >> $out/pt_c.log; tail -3 $out/pt_c.log
for v in 1 2; do HELIOS_GATHER_CTAS_PER_SM=$v timeout 600 python tools/exp_k4.py C2 20 >> $out/k4c_c2.jsonl 2>$out/k4c_c2_$v.err; done
cat $out/k4c_c2.jsonl
HELIOS_GATHER_CTAS_PER_SM=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4c_c2_flat2.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_CTAS_PER_SM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4c_c2_flat1.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
for v in 1 2; do HELIOS_GATHER_CTAS_PER_SM=$v timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bc_c2_g$v.json 2>$out/bc_c2_g$v.err; tail -c 300 $out/bc_c2_g$v.json; done
timeout 900 python bench.py > $out/bc_c3.json 2>$out/bc_c3.err; tail -c 1500 $out/bc_c3.json
timeout 900 python bench.py --zero-copy --no-cpu-baseline > $out/bc_c3_zc.json 2>$out/bc_c3_zc.err; tail -c 300 $out/bc_c3_zc.json
