# round 2: K4 VU=16 (isolated on C2 lists + pipeline), C4 green-context IO partition, C3 default.
set -x
out=${GRAFT_REPO_ROOT:-.}/gpurun_out
python -c "from paper_2310_00837_b200 import build as b; b.build(trace=False)" > /dev/null 2>&1
for v in 8 16; do HELIOS_GATHER_VU=$v timeout 600 python tools/exp_k4.py C2 20 >> $out/k4o_c2.jsonl 2>$out/k4o_c2_$v.err; done; cat $out/k4o_c2.jsonl
HELIOS_GATHER_VU=16 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4o_c2_vu16.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_VU=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gather_lists -s 70 -c 40 --csv --log-file $out/ncu_k4o_c2_vu8.csv python tools/exp_k4.py C2 1 > /dev/null 2>&1
HELIOS_GATHER_VU=16 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 3000 > $out/bo_c2_vu16.json 2>$out/bo_c2_vu16.err; tail -c 100 $out/bo_c2_vu16.json
HELIOS_GATHER_VU=16 timeout 900 python bench.py --no-cpu-baseline > $out/bo_c3_vu16.json 2>$out/bo_c3_vu16.err; tail -c 100 $out/bo_c3_vu16.json
timeout 900 python bench.py --no-cpu-baseline > $out/bo_c3.json 2>$out/bo_c3.err; tail -c 100 $out/bo_c3.json
for m in 0 16 48; do timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 40 --io-sms $m > $out/bo_c4_sm$m.json 2>$out/bo_c4_sm$m.err; tail -c 100 $out/bo_c4_sm$m.json; done
