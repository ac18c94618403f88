export CUDA_MODULE_LOADING=EAGER
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bf_c3.json 2> gpurun_out/bf_c3.err; tail -c 300 gpurun_out/bf_c3.json
timeout 900 bash tools/profile_c3.sh r01e_c3 "k_gather_lists|k_lookup"
python tools/ncu_summary.py gpurun_out/launches_r01e_c3.csv gpurun_out/prof_r01e_c3.ncu-rep > gpurun_out/ncu_r01e_c3.txt 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bf_ref.json 2> gpurun_out/bf_ref.err; cat gpurun_out/bf_ref.json | head -c 300
