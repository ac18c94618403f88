# round 2, first validation: full GPU suite, file-tier tests serialised, smoke under ncu, memcheck of the
# bad-seed paths.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -5 $out/pytest_gpu.log
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_gather.py -q -k "io_ring or three_tiers or batch_prepare or row_sizes" > $out/pytest_blocking.log 2>&1; echo "rc=$?" >> $out/pytest_blocking.log
tail -3 $out/pytest_blocking.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/ncu_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/ncu_smoke.log 2>&1; echo "rc=$?" >> $out/ncu_smoke.log
tail -3 $out/ncu_smoke.log
timeout 900 compute-sanitizer --tool memcheck --log-file $out/san_badseed.log python -m pytest tests/test_gpu_gather.py -q -k "bad_seed or seed_dtype" > $out/san_badseed.out 2>&1; echo "rc=$?" >> $out/san_badseed.out
tail -3 $out/san_badseed.out; tail -3 $out/san_badseed.log
