#!/bin/bash
# C4 column reductions: strip width x CTAs per SM x rows in flight on the final code
mkdir -p gpurun_out/col
timeout 1200 python tools/sweep_env.py colreduce 'STITCH_COL_CTAS=2,3,4,6 STITCH_COL_CT=4,8,16 STITCH_COL_U=4,8' >> gpurun_out/col/colreduce_sweep.jsonl 2>&1
echo done
