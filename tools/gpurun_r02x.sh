# round 2: programmatic dependent launch on / off, C3 (24 slots) and C2 (12 slots), two passes each, same box.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > $out/bx_c3_pdl_p$p.json 2>$out/bx_c3_pdl_p$p.err; tail -c 60 $out/bx_c3_pdl_p$p.json
  HELIOS_NO_PDL=1 timeout 900 python bench.py --no-cpu-baseline > $out/bx_c3_nopdl_p$p.json 2>$out/bx_c3_nopdl_p$p.err; tail -c 60 $out/bx_c3_nopdl_p$p.json
  timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bx_c2_pdl_p$p.json 2>$out/bx_c2_pdl_p$p.err; tail -c 60 $out/bx_c2_pdl_p$p.json
  HELIOS_NO_PDL=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bx_c2_nopdl_p$p.json 2>$out/bx_c2_nopdl_p$p.err; tail -c 60 $out/bx_c2_nopdl_p$p.json
done
HELIOS_NO_PDL=1 timeout 900 python bench.py --no-cpu-baseline --depth 32 > $out/bx_c3_nopdl_d32.json 2>$out/bx_c3_nopdl_d32.err; tail -c 60 $out/bx_c3_nopdl_d32.json
