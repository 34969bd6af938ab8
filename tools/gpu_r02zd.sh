#!/bin/bash
# model mode: 64-deep K tiles for the CUTLASS GEMMs
mkdir -p gpurun_out/gv3
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "model_mode" > gpurun_out/gv3/pytest_model.log 2>&1; echo "rc=$?" >> gpurun_out/gv3/pytest_model.log
PROBE_PRECS=tf32 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv3/gemm_variants.jsonl 2>&1
PROBE_PRECS=tf32 STITCH_GEMM_FUSED=6 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv3/gemm_variants.jsonl 2>&1
PROBE_PRECS=tf32 STITCH_GEMM_PLAIN=7 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv3/gemm_variants.jsonl 2>&1
PROBE_PRECS=tf32 STITCH_GEMM_PLAIN=6 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv3/gemm_variants.jsonl 2>&1
PROBE_PRECS=tf32 timeout 300 python tools/model_mode_probe.py >> gpurun_out/gv3/gemm_variants.jsonl 2>&1
echo done
