#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or dien" > gpurun_out/pytest_t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t.log
for gname in dien_T10 dien_T20; do timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_DIRECT_FOLD=0,1' >> gpurun_out/resident_direct.jsonl 2>&1; done
timeout 400 python tools/resident_cta_timeline.py dien_T10 > gpurun_out/resident_cta_T10_direct.txt 2>&1
echo done
