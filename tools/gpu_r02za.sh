#!/bin/bash
# model mode: CUTLASS tcgen05 TF32 GEMM configurations (plain + fused) vs cuBLASLt, tests + per-layer probe
mkdir -p gpurun_out/gv
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "model_mode" > gpurun_out/gv/pytest_model.log 2>&1; echo "rc=$?" >> gpurun_out/gv/pytest_model.log
for v in -1 0 1 2 3; do
  PROBE_PRECS=tf32 STITCH_GEMM_PLAIN=$v timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv/gemm_variants.jsonl 2>&1
done
for v in 2 3 1; do
  PROBE_PRECS=tf32 STITCH_GEMM_FUSED=$v timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv/gemm_variants.jsonl 2>&1
done
PROBE_PRECS=tf32 STITCH_GEMM_FUSED=2 STITCH_GEMM_PLAIN=2 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv/gemm_variants.jsonl 2>&1
echo done
