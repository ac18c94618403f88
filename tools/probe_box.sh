#!/bin/bash
# Step-0 probe of the GPU box: host cores, RAM, shm, disks, GPU topology.
out=${GRAFT_REPO_ROOT:-.}/gpurun_out/probe.txt
{
echo "== nproc"; nproc; python -c 'import os; print("affinity", len(os.sched_getaffinity(0)))'
echo "== lscpu"; lscpu | head -30
echo "== free"; free -g
echo "== meminfo"; head -5 /proc/meminfo
echo "== ulimit -l"; ulimit -l
echo "== df"; df -h / /tmp /dev/shm . 2>&1
echo "== lsblk"; lsblk 2>&1 | head -40
echo "== nvme"; ls -la /dev/nvme* 2>&1 | head
echo "== mounts"; mount | grep -E 'nvme|xfs|ext4|tmpfs|overlay' | head -20
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv
echo "== numa"; numactl -H 2>&1 | head; cat /sys/class/net/*/device/numa_node 2>/dev/null | head -3
echo "== torch"; python -c 'import torch;p=torch.cuda.get_device_properties(0);print(p, p.multi_processor_count)'
} > $out 2>&1
echo done
echo "== linkbench" >> $out; ./tools/linkbench >> $out 2>&1
echo "== dd" >> $out
( dd if=/dev/zero of=/tmp/ddtest bs=1M count=4096 oflag=direct 2>&1 | tail -1; dd if=/tmp/ddtest of=/dev/null bs=4k count=262144 iflag=direct 2>&1 | tail -1; dd if=/tmp/ddtest of=/dev/null bs=1M iflag=direct 2>&1 | tail -1; rm -f /tmp/ddtest ) >> $out 2>&1
