# whole-pipeline (concurrent kernels) metrics over the bench's timed NVTX range: ncu range replay
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors.sum,sm__inst_executed.sum,pcie__read_bytes.sum,sm__cycles_active.avg
for cfg in C2 C3; do
timeout 900 ncu --replay-mode app-range --nvtx --nvtx-include "timed/" --metrics $M --csv --log-file gpurun_out/range_$cfg.csv python bench.py --profile --steps 400 --warmup 5 --config $cfg > gpurun_out/range_$cfg.log 2>&1
done
cat gpurun_out/range_C2.csv | tail -20
