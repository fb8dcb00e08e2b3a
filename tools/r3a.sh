#!/bin/bash
# e2e host pipeline: PCIe copy bound (coupled vs unbounded chunks) and the
# pipeline under different slot counts / chunk sizes (ECF8_SLOTS, ECF8_CHUNK_M).
mkdir -p gpurun_out
TAG=r3a
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv,noheader
timeout 300 python tools/pcie_bound.py 2>&1 | grep -v Warn | tee gpurun_out/${TAG}_pcie.log
for cfg in "4 32" "8 32" "16 32" "8 16" "16 16" "8 64"; do
  set -- $cfg
  echo "slots=$1 chunk=$2M"
  ECF8_SLOTS=$1 ECF8_CHUNK_M=$2 timeout 300 python tools/e2e_sweep.py 2>&1 | grep layers | tee -a gpurun_out/${TAG}_e2e.log
done
ECF8_SLOTS=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host or stream or block or decompress" 2>&1 | tail -n 2
