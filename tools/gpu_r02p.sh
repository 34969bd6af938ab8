#!/bin/bash
# model mode: cuBLASLt autotune A/B + kernel names
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "model_mode" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for t in 1 8 16; do STITCH_GEMM_TUNE=$t timeout 300 python tools/model_mode_probe.py >> gpurun_out/gemm_tune.jsonl 2>&1; done
STITCH_GEMM_TUNE=8 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/gemm_launches.csv python tools/model_mode_probe.py > /dev/null 2>&1
echo done
