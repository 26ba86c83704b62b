#!/bin/bash
# run on the GPU box: tests + smoke, output into gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
