#!/bin/bash
# model mode: TMA-multicast cluster variants of the CUTLASS GEMMs
mkdir -p gpurun_out/gv2
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "model_mode" > gpurun_out/gv2/pytest_model.log 2>&1; echo "rc=$?" >> gpurun_out/gv2/pytest_model.log
for v in 3 5 -1; do
  PROBE_PRECS=tf32 STITCH_GEMM_PLAIN=$v timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv2/gemm_variants.jsonl 2>&1
done
for v in 0 4; do
  PROBE_PRECS=tf32 STITCH_GEMM_FUSED=$v timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv2/gemm_variants.jsonl 2>&1
done
echo done
