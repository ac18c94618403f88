# round 2: is the C2 step bound by DRAM bytes?  A 4 MB batch table (HELIOS_TABLE_SLOTS=262144) and an
# evict-first L2 policy on the fused gather (HELIOS_GATHER_EVICT=1), throughput and ncu range replay
# (DRAM bytes, L2 hit rate per batch) of each combination.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gather.py -x -q -k "direct" > $out/pt_aj.log 2>&1; echo "rc=$?" >> $out/pt_aj.log; tail -3 $out/pt_aj.log
HELIOS_TABLE_SLOTS=262144 HELIOS_GATHER_EVICT=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2" > $out/pt_aj2.log 2>&1; echo "rc=$?" >> $out/pt_aj2.log; tail -3 $out/pt_aj2.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,sm__inst_executed.sum
for p in 1 2; do
for v in "0 0" "262144 0" "0 1" "262144 1"; do set -- $v
  HELIOS_TABLE_SLOTS=$1 HELIOS_GATHER_EVICT=$2 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/baj_c2_t$1_e$2_p$p.json 2>/dev/null; tail -c 60 $out/baj_c2_t$1_e$2_p$p.json
done
done
for v in "0 0" "262144 0" "0 1" "262144 1"; do set -- $v
  HELIOS_TABLE_SLOTS=$1 HELIOS_GATHER_EVICT=$2 timeout 900 ncu --replay-mode app-range --nvtx --nvtx-include "timed/" --metrics $M --csv --log-file $out/range_aj_t$1_e$2.csv python bench.py --profile --steps 400 --warmup 5 --config C2 > $out/range_aj_t$1_e$2.log 2>&1
done
ls $out
