#!/bin/bash
# PCIe roofline for the e2e number: pinned H2D / D2H / both, one GPU alone and two at once
timeout 120 ./tools/nvlink_probe pcie > gpurun_out/r58_pcie_gpu0.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 120 ./tools/nvlink_probe pcie > gpurun_out/r58_pcie_pair0.jsonl 2>&1 &
CUDA_VISIBLE_DEVICES=1 timeout 120 ./tools/nvlink_probe pcie > gpurun_out/r58_pcie_pair1.jsonl 2>&1 &
wait
nvidia-smi topo -m > gpurun_out/r58_topo.txt 2>&1
nproc > gpurun_out/r58_host.txt; lscpu | head -30 >> gpurun_out/r58_host.txt; numactl -H >> gpurun_out/r58_host.txt 2>&1
true
