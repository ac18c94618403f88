# link-stream validation: plan/gather parity, then C3 default (link) vs shared-link ablation vs staged
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_gather.py -x -q > gpurun_out/pytest_link.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_link.log
tail -3 gpurun_out/pytest_link.log
for a in "" "--shared-link" "--host-staged 0.6"; do
  n=$(echo "c3$a" | tr -d ' .-')
  timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err
  tail -c 400 gpurun_out/b_$n.json
done
