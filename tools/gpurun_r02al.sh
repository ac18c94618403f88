# round 2: two-level batch table with block-window primary probing, evict-first fused gather:
# parity, then same-box A/B against the previous commit's library (HELIOS_LIB=prev) on C2 and C3.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_sample.py tests/test_gpu_gather.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py -x -q -k "not c3_full" > $out/pt_al.log 2>&1; echo "rc=$?" >> $out/pt_al.log; tail -3 $out/pt_al.log
for p in 1 2; do
for v in "prev 262144 0" "new 262144 1" "new 262144 0" "new 0 1"; do set -- $v
  L=""; [ "$1" = prev ] && L=prev
  HELIOS_LIB=$L HELIOS_TABLE_SLOTS=$2 HELIOS_GATHER_EVICT=$3 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bal_c2_$1_t$2_e$3_p$p.json 2>/dev/null; tail -c 60 $out/bal_c2_$1_t$2_e$3_p$p.json
done
done
for v in "prev 262144" "new 262144" "prev 262144" "new 262144"; do set -- $v
  L=""; [ "$1" = prev ] && L=prev
  HELIOS_LIB=$L HELIOS_TABLE_SLOTS=$2 timeout 900 python bench.py --no-cpu-baseline --steps 1500 >> $out/bal_c3_$1.jsonl 2>/dev/null; tail -c 60 $out/bal_c3_$1.jsonl
done
