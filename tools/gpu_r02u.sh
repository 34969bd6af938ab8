#!/bin/bash
# sanitizers on the final resident template (W-warp fold, direct fold, restricted waits)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident" > gpurun_out/memcheck_resident.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident_template_matches" > gpurun_out/racecheck_resident.log 2>&1
timeout 1500 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident_template_matches" > gpurun_out/synccheck_resident.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "bert_layer or shard_plans" > gpurun_out/memcheck_layer_shards.log 2>&1
tail -n 2 gpurun_out/memcheck_resident.log gpurun_out/racecheck_resident.log gpurun_out/synccheck_resident.log gpurun_out/memcheck_layer_shards.log
