# round 2: K4 (fused HBM-only gather) alone on C2's real lists with the evict-first policy: grid / loads-in-
# flight sweep (CUDA events), then ncu kernel-only durations and one full capture of the fastest setting.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
for v in "4 1" "4 2" "4 3" "8 1" "8 2" "8 3" "16 1"; do set -- $v
  HELIOS_GATHER_VU=$1 HELIOS_GATHER_CTAS_PER_SM=$2 timeout 600 python tools/exp_k4.py C2 20 2>/dev/null | sed "s/^/{\"vu\": $1, \"per_sm\": $2, \"r\": /; s/$/}/" >> $out/k4aq.jsonl
done
cat $out/k4aq.jsonl
for v in "8 2" "4 3" "4 1"; do set -- $v
  HELIOS_GATHER_VU=$1 HELIOS_GATHER_CTAS_PER_SM=$2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gather_direct -c 40 --csv --log-file $out/ncu_k4aq_vu$1_s$2.csv python tools/exp_k4.py C2 1 > $out/ncu_k4aq_vu$1_s$2.log 2>&1
done
HELIOS_GATHER_VU=8 HELIOS_GATHER_CTAS_PER_SM=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_direct -s 20 -c 1 -o $out/prof_k4aq python tools/exp_k4.py C2 1 > $out/ncu_full_k4aq.log 2>&1
timeout 600 python tools/exp_split.py C2 > $out/split_aq.json 2>/dev/null; cat $out/split_aq.json
ls $out
