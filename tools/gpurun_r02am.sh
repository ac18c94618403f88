# round 2: adaptive home region of the batch table (keys homed in 2^k >= 2.5 n_L(prev batch) slots, probing
# on through the worst-case table) + evict-first fused gather: parity, then same-box A/B against the previous
# commit's library (HELIOS_LIB=prev) on C2 and C3.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_sample.py tests/test_gpu_gather.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py -x -q -k "not c3_full" > $out/pt_am.log 2>&1; echo "rc=$?" >> $out/pt_am.log; tail -3 $out/pt_am.log
for p in 1 2; do
for v in "prev x 0" "new x 1" "new 0 1" "new x 0"; do set -- $v
  L=""; [ "$1" = prev ] && L=prev
  H=""; [ "$2" != x ] && H=$2
  env ${L:+HELIOS_LIB=$L} ${H:+HELIOS_TABLE_HOME=$H} HELIOS_GATHER_EVICT=$3 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bam_c2_$1_h$2_e$3_p$p.json 2>/dev/null; tail -c 60 $out/bam_c2_$1_h$2_e$3_p$p.json
done
done
for v in prev new prev new; do
  env ${v/new/} $( [ $v = prev ] && echo HELIOS_LIB=prev ) timeout 900 python bench.py --no-cpu-baseline --steps 1500 >> $out/bam_c3_$v.jsonl 2>/dev/null; tail -c 60 $out/bam_c3_$v.jsonl
done
