#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or dien" > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
for gname in dien_T10 dien_T20; do timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_INLINE=1,0' >> gpurun_out/resident_inline.jsonl 2>&1; done
timeout 400 python tools/resident_cta_timeline.py dien_T10 > gpurun_out/resident_cta_T10_noinline.txt 2>&1
echo done
