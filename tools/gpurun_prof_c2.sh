export CUDA_MODULE_LOADING=EAGER
bash tools/profile_c3.sh r01e_c2 "k_fill_insert|k_dedup_assign|k_count_scan|k_gather_lists|k_lookup|k_table_clear|k_relabel" --config C2
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -c 13 -o gpurun_out/prof_r01e_c2all python bench.py --profile --steps 3 --warmup 3 --config C2 > gpurun_out/ncu_full_c2all.log 2>&1
ls -la gpurun_out/*.ncu-rep
