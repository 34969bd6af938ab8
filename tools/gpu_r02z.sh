#!/bin/bash
# (1) model mode: CUTLASS stream-K GEMM for ffn2 vs cuBLASLt; (2) per-team TMA rings (STITCH_STAGE=2):
# parity tests, A/B against the register pipeline and the per-CTA tile ring; (3) sanitizers
mkdir -p gpurun_out/team
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "model_mode" > gpurun_out/team/pytest_model.log 2>&1; echo "rc=$?" >> gpurun_out/team/pytest_model.log
for sk in 0 1; do for sp in 0 2 3 4; do [ $sk = 0 ] && [ $sp != 0 ] && continue
  PROBE_PRECS=tf32 STITCH_GEMM_SK=$sk STITCH_GEMM_SK_SPLITS=$sp timeout 300 python tools/model_mode_probe.py >> gpurun_out/team/model_sk.jsonl 2>&1
done; done
PROBE_PRECS=tf32 timeout 300 python tools/model_mode_probe.py >> gpurun_out/team/model_sk_auto.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_exec.py -q -x -k "tma_staged" > gpurun_out/team/pytest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/team/pytest_tma.log
for gr in ln_4096x768 bert_resln attn_softmax bert_cut; do
  timeout 600 python tools/sweep_env.py $gr 'STITCH_STAGE=0,1,2 STITCH_STAGES=2,3,4' >> gpurun_out/team/sweep.jsonl 2>&1
done
timeout 600 python tools/sweep_env.py ln_4096x768 'STITCH_STAGE=2 STITCH_STAGES=4,6,8 STITCH_STAGE_SMEM_KB=110,200' >> gpurun_out/team/sweep_deep.jsonl 2>&1
timeout 600 python tools/sweep_env.py bert_resln 'STITCH_STAGE=2 STITCH_STAGES=2,3,4 STITCH_STAGE_SMEM_KB=110,200' >> gpurun_out/team/sweep_deep.jsonl 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x -k "streamk" > gpurun_out/team/memcheck_sk.log 2>&1; echo "rc=$?" >> gpurun_out/team/memcheck_sk.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
    -k "tma_staged and (ln_4096 or bert_resln or many_short or smem_team)" > gpurun_out/team/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/team/racecheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x \
    -k "tma_staged and (ln_4096 or bert_resln or many_short or smem_team)" > gpurun_out/team/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/team/memcheck.log
echo done
