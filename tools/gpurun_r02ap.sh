# round 2: evict-last L2 policy on the batch-table accesses (A/B build libhelios_tel.so, HELIOS_LIB=tel):
# sampler parity with it, then C2 / C3 A/B on one box against the default build.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
HELIOS_LIB=tel timeout 1200 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py -x -q -k "not c3_full and not c3_scaled" > $out/pt_ap.log 2>&1; echo "rc=$?" >> $out/pt_ap.log; tail -3 $out/pt_ap.log
for p in 1 2; do
for v in def tel; do
  L=""; [ $v = tel ] && L=tel
  env ${L:+HELIOS_LIB=$L} timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bap_c2_${v}_p$p.json 2>/dev/null; tail -c 60 $out/bap_c2_${v}_p$p.json
done
done
for p in 1 2; do
for v in def tel; do
  L=""; [ $v = tel ] && L=tel
  env ${L:+HELIOS_LIB=$L} timeout 900 python bench.py --no-cpu-baseline --steps 1500 > $out/bap_c3_${v}_p$p.json 2>/dev/null; tail -c 60 $out/bap_c3_${v}_p$p.json
done
done
