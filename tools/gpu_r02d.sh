#!/bin/bash
# resident template: parity tests + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or persistent" > gpurun_out/pytest_resident.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_resident.log
for g in dien_T10 dien_T20; do
  timeout 300 python tools/sweep_env.py $g 'STITCH_RESIDENT=0,1' >> gpurun_out/resident_ab.jsonl 2>&1
done
echo done
