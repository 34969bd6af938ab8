#!/bin/bash
# validate + measure: resident split groups (fillers), batched grid placeholders, TMA 2 stages
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or dien or bert_layer or tma or opaque or model_mode or refined" > gpurun_out/pytest_n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.log
for gname in dien_T10 dien_T20; do
  timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_FILL=0,3,6' >> gpurun_out/resident_fill.jsonl 2>&1
done
timeout 300 python tools/resident_timeline.py dien_T10 > gpurun_out/resident_timeline_fill3.txt 2>&1
timeout 600 python tools/sweep_env.py bert_layer 'STITCH_OPAQUE_GRID_BATCH=0,4,8,12' > gpurun_out/grid_batch.jsonl 2>&1
timeout 400 python tools/sweep_env.py ln_4096x768 'STITCH_STAGE=1' 'STITCH_STAGES=2' > gpurun_out/tma2.jsonl 2>&1
echo done
