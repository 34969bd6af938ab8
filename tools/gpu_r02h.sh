#!/bin/bash
# balanced regional CTA sizing (k CTAs per SM) with serial / one-call latency
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "config or fixture or edge or regional or row or resident" > gpurun_out/pytest_rows2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows2.log
for g in ln_4096x768 bert_resln ln2pass_4096x768; do
  timeout 600 python tools/sweep_env.py $g 'STITCH_ROW_CTAS_PER_SM=0,1,2,3,4' >> gpurun_out/rows_k_sweep.jsonl 2>&1
done
timeout 600 python tools/sweep_env.py colreduce 'STITCH_COL_CTAS=2,3' 'STITCH_COL_CT=4,8,16' >> gpurun_out/rows_k_sweep.jsonl 2>&1
echo done
