#!/bin/bash
# bert_cut (C3 headline) packing knobs: local unroll x local CTAs/SM x body order, CTA size
mkdir -p gpurun_out
timeout 1500 python tools/sweep_env.py bert_cut 'STITCH_LOCAL_U=2,4' 'STITCH_LOCAL_CTAS=9,18,32' 'STITCH_BODY_ORDER=0,1' > gpurun_out/bert_cut_sweep.jsonl 2>&1
timeout 400 python tools/sweep_env.py bert_cut 'STITCH_ROW_BLOCK=128,256' 'STITCH_LOCAL_U=2,4' >> gpurun_out/bert_cut_sweep.jsonl 2>&1
timeout 300 python tools/sweep_env.py bert_gelu 'STITCH_LOCAL_U=2,4' >> gpurun_out/bert_cut_sweep.jsonl 2>&1
echo done
