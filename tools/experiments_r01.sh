#!/bin/bash
# How the round-1 experiment files under profiles/ were produced (run on the GPU box via gpurun from
# the repo root; each bench line is one JSON object).  Sections can be run separately:
#   bash tools/experiments_r01.sh <section>
set -u
run() { n=$1; shift; timeout 400 env "$@" > gpurun_out/exp_$n.json 2> gpurun_out/exp_$n.err; }
B="python bench.py --no-cpu-baseline --parity-batches 1"
case "${1:-}" in
  link)      # link_ablation_r01.jsonl: link stream vs per-slot gather, depth, PDL
    run link1 $B --link-stream --depth 6; run shared $B --depth 6
    run link2 HELIOS_PLAN_LINKS=2 $B --link-stream --depth 6; run link3 HELIOS_PLAN_LINKS=3 $B --link-stream --depth 6
    run st_shared $B --host-staged 0.6 --depth 6
    for d in 6 8 12 16; do run c2d$d $B --config C2 --depth $d; done
    run c2nopdl HELIOS_NO_PDL=1 $B --config C2 --depth 6 ;;
  grid)      # gather_grid_r01.jsonl: K4 grid / host-warp sweeps were run with temporary env knobs
    run c3 $B; run c2 $B --config C2 ;;
  hostlink)  # hostorder_r01.jsonl, hostnoise_r01.jsonl, iotlb_r01.jsonl, host_slots_r01.json, layout_r01.json
    export CUDA_MODULE_LOADING=EAGER
    python tools/host_slots.py /tmp/c3s 96 > gpurun_out/host_slots.json
    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/hostorder tools/hostorder.cu && /tmp/hostorder /tmp/c3s 99900000 512 > gpurun_out/hostorder.jsonl
    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/hostnoise tools/hostnoise.cu && /tmp/hostnoise /tmp/c3s 99900000 512 148 > gpurun_out/hostnoise.jsonl
    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/iotlb tools/iotlb.cu && /tmp/iotlb 51 > gpurun_out/iotlb.jsonl
    python tools/layout_study.py 1.0 32 > gpurun_out/layout.json ;;
  sectors)   # sectorbench_r01.jsonl
    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sb tools/sectorbench.cu && /tmp/sb > gpurun_out/sectorbench.jsonl ;;
  range)     # ncu_range_r01e.json: counters over the whole pipelined timed region (all concurrent kernels)
    M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__inst_executed.sum,pcie__read_bytes.sum
    for cfg in C2 C3; do
      ncu --replay-mode app-range --nvtx --nvtx-include "timed/" --metrics $M --csv --log-file gpurun_out/range_$cfg.csv \
          python bench.py --profile --steps 400 --warmup 5 --config $cfg
    done ;;
  ncu)       # ncu_r01f_*.txt, ncu_launches_r01f_*.csv, ncu_traffic_r01.json
    bash tools/profile_c3.sh r01f_c3 "k_gather_lists|k_lookup"
    bash tools/profile_c3.sh r01f_c2 "k_gather_lists|k_lookup" --config C2 ;;
  *) echo "sections: link grid hostlink sectors range ncu" ;;
esac
