#!/bin/bash
# ncu evidence for the bench's timed region (B200_PROFILING.md recipe): launch list + one full capture
# of the dominant kernels.  Usage: tools/profile_c3.sh <tag> <kernel-regex> [bench args...]
tag=$1; shift
kre=$1; shift
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv \
    --log-file $out/launches_$tag.csv python bench.py --profile --steps 5 --warmup 3 "$@" > $out/ncu_launch_$tag.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"$kre" -c 6 -o $out/prof_$tag python bench.py --profile --steps 3 --warmup 3 "$@" > $out/ncu_full_$tag.log 2>&1
echo done
