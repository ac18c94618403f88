# round 2: IO-kernel ncu evidence (C1, C4), compute-sanitizer synccheck / initcheck, flat-K4 STG stores,
# C4 host tier on/off at one scale, C3 depth / stager variants.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_io|k_gather_lists|k_lookup" -c 60 --csv --log-file $out/ncu_io_c1.csv python bench.py --config C1 --profile --steps 20 --warmup 3 --no-cpu-baseline > $out/ncu_io_c1.log 2>&1; echo "rc=$?" >> $out/ncu_io_c1.log
timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_io|k_gather_lists|k_lookup" -c 30 --csv --log-file $out/ncu_io_c4.csv python bench.py --config C4 --scale 0.02 --profile --steps 6 --warmup 3 --no-cpu-baseline > $out/ncu_io_c4.log 2>&1; echo "rc=$?" >> $out/ncu_io_c4.log
mkdir -p $out/san
timeout 1200 compute-sanitizer --tool synccheck --log-file $out/san/synccheck.log python -m pytest tests/test_gpu_gather.py tests/test_gpu_sample.py -q -x -k "three_tiers_c1 and False-True-1.0-0.6 or io_ring or medium_graph and chain and 1024" > $out/san/synccheck.out 2>&1; echo "rc=$?" >> $out/san/synccheck.out; tail -3 $out/san/synccheck.log
timeout 1200 compute-sanitizer --tool initcheck --log-file $out/san/initcheck.log python -m pytest tests/test_gpu_gather.py tests/test_gpu_sample.py -q -x -k "three_tiers_c1 and False-True-1.0-0.6 or io_ring or medium_graph and chain and 1024" > $out/san/initcheck.out 2>&1; echo "rc=$?" >> $out/san/initcheck.out; tail -3 $out/san/initcheck.log
timeout 900 compute-sanitizer --tool memcheck --log-file $out/san/memcheck_tiled_groups.log python -m pytest tests/test_gpu_plan.py tests/test_gpu_sample.py -q -x -k "groups_c1_epoch and 2-2 or medium_graph and tiled and 1024 or green" > $out/san/memcheck_tiled_groups.out 2>&1; echo "rc=$?" >> $out/san/memcheck_tiled_groups.out; tail -3 $out/san/memcheck_tiled_groups.log
timeout 600 python tools/exp_k4.py C2 20 > $out/k4q_c2.jsonl 2>$out/k4q.err; cat $out/k4q_c2.jsonl
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bq_c2.json 2>$out/bq_c2.err; tail -c 100 $out/bq_c2.json
for h in 0.4 0; do timeout 900 python bench.py --config C4 --scale 0.02 --no-cpu-baseline --steps 40 --host-frac $h > $out/bq_c4_s002_host$h.json 2>$out/bq_c4_s002_host$h.err; tail -c 100 $out/bq_c4_s002_host$h.json; done
timeout 900 python bench.py --no-cpu-baseline --depth 16 > $out/bq_c3_d16.json 2>$out/bq_c3_d16.err; tail -c 100 $out/bq_c3_d16.json
for w in 12 16; do timeout 900 python bench.py --no-cpu-baseline --stage-workers $w > $out/bq_c3_w$w.json 2>$out/bq_c3_w$w.err; tail -c 100 $out/bq_c3_w$w.json; done
