# round 2: staged fix (relaxed claim loads), cluster sampler modes, link probe sweep.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
timeout 1800 python -m pytest tests/test_gpu_sample.py tests/test_gpu_gather.py tests/test_gpu_plan.py tests/test_gpu_fullsize.py -x -q > $out/pt_d.log 2>&1; echo "rc=$?" >> $out/pt_d.log; tail -3 $out/pt_d.log
timeout 900 python bench.py --no-cpu-baseline > $out/bd_c3.json 2>$out/bd_c3.err; tail -c 300 $out/bd_c3.json
for m in chain cluster cluster16; do HELIOS_SAMPLE_MODE=$m timeout 600 python tools/exp_split.py C2 > $out/split_d_$m.json 2>$out/split_d_$m.err; cat $out/split_d_$m.json; done
for m in cluster cluster16; do HELIOS_SAMPLE_MODE=$m timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bd_c2_$m.json 2>$out/bd_c2_$m.err; tail -c 200 $out/bd_c2_$m.json; done
HELIOS_SAMPLE_MODE=cluster timeout 900 python bench.py --no-cpu-baseline > $out/bd_c3_cluster.json 2>$out/bd_c3_cluster.err; tail -c 200 $out/bd_c3_cluster.json
