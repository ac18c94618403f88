# round 2 validation of the new defaults (split host-row kernel, depth 24 with a host tier): full GPU
# suite, smoke, default bench (C3) + C2, ncu launch list + full capture, whole-pipeline range replay.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $out/build_t.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pt_t.log 2>&1; echo "rc=$?" >> $out/pt_t.log; tail -3 $out/pt_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_t.log 2>&1; echo "rc=$?" >> $out/smoke_t.log; tail -2 $out/smoke_t.log
timeout 900 python bench.py > $out/bt_c3.json 2>$out/bt_c3.err; tail -c 200 $out/bt_c3.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bt_c2.json 2>$out/bt_c2.err; tail -c 100 $out/bt_c2.json
timeout 900 python bench.py --no-cpu-baseline --depth 32 > $out/bt_c3_d32.json 2>$out/bt_c3_d32.err; tail -c 100 $out/bt_c3_d32.json
timeout 1200 bash tools/profile_c3.sh r02t_c3 "k_gather_lists|k_gather_host|k_lookup" > /dev/null 2>&1
timeout 900 bash tools/profile_c3.sh r02t_c2 "k_gather_lists|k_lookup" --config C2 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__inst_executed.sum,pcie__read_bytes.sum
for cfg in C2 C3; do
  timeout 1200 ncu --replay-mode app-range --nvtx --nvtx-include "timed/" --metrics $M --csv --log-file $out/range_t_$cfg.csv python bench.py --profile --steps 400 --warmup 5 --config $cfg > $out/range_t_$cfg.log 2>&1
done
ls -la $out
