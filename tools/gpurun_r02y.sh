# round 2: device pipeline trace (traced build) of C2 at 12 slots and C3 at 24 slots with the current kernels.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python tools/trace_pipeline.py C2 12 > $out/trace_y_c2.json 2>$out/trace_y_c2.err; tail -c 1500 $out/trace_y_c2.json
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 1200 python tools/trace_pipeline.py C3 24 > $out/trace_y_c3.json 2>$out/trace_y_c3.err; tail -c 1500 $out/trace_y_c3.json
