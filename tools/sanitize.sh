#!/bin/bash
# compute-sanitizer passes over the generated kernels (run under gpurun):
# memcheck (out-of-bounds / misaligned), racecheck (shared-memory hazards),
# synccheck (barrier misuse).  Summaries land in gpurun_out/.
# The second group covers the north-star variants: TMA-staged regional rows
# (STITCH_STAGE=1, cp.async.bulk + mbarrier ring) and the cooperative
# grid-barrier global template (STITCH_COL_SYNC=grid), plus the multi-domain
# row bodies and dotted tensor names.
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "edge_shapes or op_and_dtype or (fixture_parity and stitched) or dag or low_level" > gpurun_out/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "edge_shapes or softmax or layernorm or variance" > gpurun_out/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "edge_shapes" > gpurun_out/synccheck.log 2>&1
V="tma_staged or grid_barrier or dotted or (config_parity_full_size and dien and 1)"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "$V" > gpurun_out/memcheck_variants.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "tma_staged or grid_barrier" > gpurun_out/racecheck_variants.log 2>&1
timeout 1500 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "tma_staged or grid_barrier" > gpurun_out/synccheck_variants.log 2>&1
# resident template (one cluster kernel: DSMEM st.async pushes, mbarriers,
# cp.async.bulk parameter staging, split placeholder groups)
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident" > gpurun_out/memcheck_resident.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident_template_matches" > gpurun_out/racecheck_resident.log 2>&1
timeout 1500 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "resident_template_matches" > gpurun_out/synccheck_resident.log 2>&1
# model mode (cuBLASLt GEMMs in the graph), BERT layer, shard plans, host paths
timeout 2000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exec.py -q -x \
  -k "bert_layer or shard_plans or refined or model_mode or two_rank or chunked" > gpurun_out/memcheck_layer_shards.log 2>&1
tail -n 2 gpurun_out/memcheck*.log gpurun_out/racecheck*.log gpurun_out/synccheck*.log
