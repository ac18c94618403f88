set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -c 600 gpurun_out/b_c3.json
timeout 600 python bench.py --serial-gather 1 --no-cpu-baseline > gpurun_out/b_c3_serial.json 2> gpurun_out/b_c3_serial.err; tail -c 300 gpurun_out/b_c3_serial.json
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/b_c2.json 2>gpurun_out/b_c2.err
timeout 600 python bench.py --config C2 --serial-gather 1 --no-cpu-baseline > gpurun_out/b_c2_serial.json 2>gpurun_out/b_c2_serial.err
