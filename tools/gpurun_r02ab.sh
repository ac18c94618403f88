# round 2: K4 register footprint (VU 2 / 4) x fill CTAs per SM (2 / 4) on C2, same box; C3 with VU 4.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HELIOS_GATHER_VU=2 timeout 600 python -m pytest tests/test_gpu_gather.py -x -q -k "three_tiers or row_sizes" > $out/pt_ab.log 2>&1; echo "rc=$?" >> $out/pt_ab.log; tail -2 $out/pt_ab.log
for vu in 2 4 8; do for fc in 2 4; do
  HELIOS_GATHER_VU=$vu HELIOS_FILL_CTAS_PER_SM=$fc timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bab_c2_vu${vu}_f$fc.json 2>/dev/null; tail -c 60 $out/bab_c2_vu${vu}_f$fc.json
done; done
HELIOS_GATHER_VU=4 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --depth 16 > $out/bab_c2_vu4_d16.json 2>/dev/null; tail -c 60 $out/bab_c2_vu4_d16.json
HELIOS_GATHER_VU=2 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 --depth 16 > $out/bab_c2_vu2_d16.json 2>/dev/null; tail -c 60 $out/bab_c2_vu2_d16.json
for vu in 4 8; do HELIOS_GATHER_VU=$vu timeout 900 python bench.py --no-cpu-baseline > $out/bab_c3_vu$vu.json 2>/dev/null; tail -c 60 $out/bab_c3_vu$vu.json; done
