#!/bin/bash
# packed row team width: full GPU suite + bert_cut knobs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep_env.py bert_cut 'STITCH_PACKED_ROW_NJ=1,2' 'STITCH_LOCAL_CTAS=0,4,6,12' > gpurun_out/cut_nj2.jsonl 2>&1
echo done
