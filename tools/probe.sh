#!/bin/bash
# First GPU call: machine facts + host-link microbenchmark.
set -x
mkdir -p gpurun_out
{
  nproc; lscpu | head -20; free -g; cat /proc/meminfo | head -5
  nvidia-smi; nvidia-smi topo -m
  nvidia-smi -q | grep -A12 -i "PCI$" | head -40
  nvidia-smi -q | grep -i -A3 "Link Width\|Link Gen\|GPU Link Info" | head -40
  ulimit -l
} > gpurun_out/probe_sys.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/probe_hostlink.cu
timeout 300 /tmp/probe 4096 32768 > gpurun_out/probe_hostlink.txt 2>&1
echo "exit=$?" >> gpurun_out/probe_hostlink.txt
cat gpurun_out/probe_hostlink.txt | tail -5
