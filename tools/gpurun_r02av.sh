# round 2 final validation (fill <= 4 CTAs per SM, C2 depth 16, adaptive table home, evict-first policies):
# full GPU suite, smoke, default bench (C3) + C2 + C4 + C1, ncu launch lists and full captures, range replay.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $out/build_av.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pt_av.log 2>&1; echo "rc=$?" >> $out/pt_av.log; tail -3 $out/pt_av.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_av.log 2>&1; echo "rc=$?" >> $out/smoke_av.log; tail -2 $out/smoke_av.log
timeout 900 python bench.py > $out/bav_c3.json 2>$out/bav_c3.err; tail -c 200 $out/bav_c3.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bav_c2.json 2>$out/bav_c2.err; tail -c 100 $out/bav_c2.json
timeout 900 python bench.py --config C4 --no-cpu-baseline > $out/bav_c4.json 2>$out/bav_c4.err; tail -c 100 $out/bav_c4.json
timeout 600 python bench.py --config C1 --no-cpu-baseline > $out/bav_c1.json 2>$out/bav_c1.err; tail -c 100 $out/bav_c1.json
timeout 1200 bash tools/profile_c3.sh ao_c3 "k_gather_lists|k_gather_host|k_lookup" > /dev/null 2>&1
timeout 900 bash tools/profile_c3.sh ao_c2 "k_gather_direct|k_fill_seg" --config C2 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__inst_executed.sum,pcie__read_bytes.sum
for cfg in C2 C3; do
  timeout 1200 ncu --replay-mode app-range --nvtx --nvtx-include "timed/" --metrics $M --csv --log-file $out/range_av_$cfg.csv python bench.py --profile --steps 400 --warmup 5 --config $cfg > $out/range_av_$cfg.log 2>&1
done
ls -la $out
