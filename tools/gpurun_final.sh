# Round-end validation on one B200: full GPU suite, smoke, the default bench line (C3, with the CPU
# oracle baseline), C2, and the reference arm.  Outputs land in gpurun_out/.
export CUDA_MODULE_LOADING=EAGER
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bf_c3.json 2> gpurun_out/bf_c3.err; tail -c 300 gpurun_out/bf_c3.json
timeout 600 python bench.py --config C2 > gpurun_out/bf_c2.json 2> gpurun_out/bf_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bf_ref.json 2> gpurun_out/bf_ref.err; head -c 200 gpurun_out/bf_ref.json
