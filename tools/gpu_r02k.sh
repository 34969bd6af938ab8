#!/bin/bash
# TMA-staged regional rows vs the register pipeline, current code (3 timings)
mkdir -p gpurun_out
for gname in ln_4096x768 bert_resln attn_softmax ln2pass_4096x768; do
  timeout 400 python tools/sweep_env.py $gname 'STITCH_STAGE=0' >> gpurun_out/tma_vs_reg.jsonl 2>&1
  timeout 600 python tools/sweep_env.py $gname 'STITCH_STAGE=1' 'STITCH_STAGES=2,3,4,6' >> gpurun_out/tma_vs_reg.jsonl 2>&1
done
echo done
