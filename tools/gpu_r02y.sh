#!/bin/bash
# model mode: CUTLASS tcgen05 GEMM with fused bias + GELU epilogue
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "model_mode or fused_gemm or refined" > gpurun_out/pytest_y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.log
for f in 0 1; do STITCH_GEMM_FUSE=$f timeout 300 python tools/model_mode_probe.py 2>&1 | head -1 >> gpurun_out/gemm_fuse.jsonl; done
timeout 600 python tools/sweep_env.py bert_layer 'STITCH_GEMM_FUSE=0,1' > /dev/null 2>&1
STITCH_GEMM_FUSE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/gemm_fuse_launches.csv python tools/model_mode_probe.py > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -k "fused_gemm or (model_mode and tf32)" > gpurun_out/memcheck_fused_gemm.log 2>&1
tail -n 2 gpurun_out/memcheck_fused_gemm.log
echo done
