#!/bin/bash
# Host side of the e2e path on the GPU box: topology, host write bandwidth, rl_label_into variants.
mkdir -p gpurun_out
{ lscpu | head -25; numactl --hardware 2>&1 | head -12; nvidia-smi topo -m 2>&1 | head -8; cat /sys/fs/cgroup/cpuset.cpus.effective 2>/dev/null; nproc; } > gpurun_out/hp_topo.txt 2>&1
g++ -O3 -pthread tools/host_bw.cpp -o /tmp/host_bw && /tmp/host_bw > gpurun_out/hp_bw.txt 2>&1
python tools/e2e_probe.py --variants "base;OUT=fill;OUT=comps;OUT=none" --steps 5 > gpurun_out/hp_e2e.txt 2>&1
RUNLAB_GPU_DEBUG_TIMELINE=1 python tools/e2e_probe.py --variants "base" --steps 1 > gpurun_out/hp_tl.txt 2>&1
