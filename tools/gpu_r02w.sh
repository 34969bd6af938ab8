#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or dien" > gpurun_out/pytest_w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.log
for gname in dien_T10 dien_T20; do timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_LOOP=0,1' >> gpurun_out/resident_loop.jsonl 2>&1; done
timeout 400 python tools/resident_cta_timeline.py dien_T10 > gpurun_out/resident_cta_T10_loop.txt 2>&1
STITCH_RESIDENT=1 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -c 2 -o gpurun_out/dien_res_loop -f python tools/ncu_target.py dien_T10 > gpurun_out/ncu_dien_loop.log 2>&1
echo done
