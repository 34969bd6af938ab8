#!/bin/bash
# regional rows: shared-memory broadcast hoist (no spill) + CTA-size sweep with
# device-side one-call latency
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "config or fixture or edge or regional or row" > gpurun_out/pytest_rows.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows.log
for g in bert_resln ln_4096x768; do
  timeout 600 python tools/sweep_env.py $g 'STITCH_ROW_HOIST_BCAST=1,2' 'STITCH_ROW_BLOCK=0,224,448' >> gpurun_out/rows_sweep.jsonl 2>&1
done
timeout 300 python tools/sweep_env.py ln2pass_4096x768 'STITCH_ROW_BLOCK=0,224,448' >> gpurun_out/rows_sweep.jsonl 2>&1
for g in bert_cut attn_softmax colreduce bert_gelu; do
  timeout 300 python tools/sweep_env.py $g >> gpurun_out/rows_sweep.jsonl 2>&1
done
echo done
