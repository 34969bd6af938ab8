#!/bin/bash
# model mode: CUTLASS GEMMs under programmatic dependent launch (STITCH_GEMM_PDL)
mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "model_mode" > gpurun_out/pdl/pytest_model.log 2>&1; echo "rc=$?" >> gpurun_out/pdl/pytest_model.log
for p in 0 1 0 1; do
  PROBE_PRECS=tf32 STITCH_GEMM_PDL=$p timeout 300 python tools/model_mode_probe.py >> gpurun_out/pdl/gemm_pdl.jsonl 2>&1
done
echo done
