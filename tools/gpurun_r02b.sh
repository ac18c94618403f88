# round 2: K4 flat mapping vs bulk-copy (TMA engine) variant, isolated on real C2 lists + pipeline benches.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_plan.py -x -q > $out/pt_b.log 2>&1; echo "rc=$?" >> $out/pt_b.log; tail -2 $out/pt_b.log
HELIOS_GATHER_BULK=1 timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_fullsize.py -x -q -k "not c3_full" > $out/pt_b_bulk.log 2>&1; echo "rc=$?" >> $out/pt_b_bulk.log; tail -2 $out/pt_b_bulk.log
for v in 1 2 4; do HELIOS_GATHER_CTAS_PER_SM=$v timeout 600 python tools/exp_k4.py C2 20 >> $out/k4_c2.jsonl 2>$out/k4_c2_$v.err; done
HELIOS_GATHER_BULK=1 timeout 600 python tools/exp_k4.py C2 20 >> $out/k4_c2.jsonl 2>$out/k4_c2_bulk.err
cat $out/k4_c2.jsonl
HELIOS_GATHER_CTAS_PER_SM=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4_c2_flat.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_BULK=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4_c2_bulk.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_CTAS_PER_SM=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_lists -s 70 -c 2 -o $out/prof_k4_c2_flat python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_BULK=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_lists -s 70 -c 2 -o $out/prof_k4_c2_bulk python tools/exp_k4.py C2 1 > /dev/null 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 2000 > $out/b_c2.json 2>$out/b_c2.err; tail -c 400 $out/b_c2.json
HELIOS_GATHER_BULK=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 2000 > $out/b_c2_bulk.json 2>$out/b_c2_bulk.err; tail -c 400 $out/b_c2_bulk.json
timeout 900 python bench.py --no-cpu-baseline > $out/b_c3.json 2>$out/b_c3.err; tail -c 400 $out/b_c3.json
