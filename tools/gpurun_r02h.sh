set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pt_h.log 2>&1; echo "rc=$?" >> $out/pt_h.log; tail -3 $out/pt_h.log
timeout 900 python bench.py > $out/bh_c3.json 2>$out/bh_c3.err; tail -c 200 $out/bh_c3.json
timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bh_c2.json 2>$out/bh_c2.err
