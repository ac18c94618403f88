# round 2: why e2e trails value on C3 at 24 slots: one whole-batch graph vs the two half graphs, PDL off;
# plus the N>1 bench path (2 ranks on one GPU, gloo) on C2 and C3.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --no-cpu-baseline > $out/bw_c3.json 2>$out/bw_c3.err; tail -c 60 $out/bw_c3.json
HELIOS_PLAN_TWO_GRAPHS=1 timeout 900 python bench.py --no-cpu-baseline > $out/bw_c3_2g.json 2>$out/bw_c3_2g.err; tail -c 60 $out/bw_c3_2g.json
HELIOS_NO_PDL=1 timeout 900 python bench.py --no-cpu-baseline > $out/bw_c3_nopdl.json 2>$out/bw_c3_nopdl.err; tail -c 60 $out/bw_c3_nopdl.json
HELIOS_PLAN_TWO_GRAPHS=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bw_c2_2g.json 2>$out/bw_c2_2g.err; tail -c 60 $out/bw_c2_2g.json
HELIOS_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config C2 --steps 1000 --warmup 5 --no-cpu-baseline > $out/bw_c2_n2.json 2>$out/bw_c2_n2.err; tail -c 300 $out/bw_c2_n2.json
HELIOS_BENCH_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 1000 --warmup 5 --no-cpu-baseline > $out/bw_c3_n2.json 2>$out/bw_c3_n2.err; tail -c 300 $out/bw_c3_n2.json
HELIOS_BENCH_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1000 --warmup 5 --no-cpu-baseline --hbm-replicated > $out/bw_c3_n2_rep.json 2>$out/bw_c3_n2_rep.err; tail -c 300 $out/bw_c3_n2_rep.json
