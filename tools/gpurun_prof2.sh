export CUDA_MODULE_LOADING=EAGER
timeout 900 bash tools/profile_c3.sh r01f_c3 "k_gather_lists|k_lookup"
timeout 600 bash tools/profile_c3.sh r01f_c2 "k_gather_lists|k_lookup" --config C2
python tools/ncu_summary.py gpurun_out/launches_r01f_c3.csv gpurun_out/prof_r01f_c3.ncu-rep > gpurun_out/ncu_r01f_c3.txt 2>&1
python tools/ncu_summary.py gpurun_out/launches_r01f_c2.csv gpurun_out/prof_r01f_c2.ncu-rep > gpurun_out/ncu_r01f_c2.txt 2>&1
head -12 gpurun_out/ncu_r01f_c3.txt
