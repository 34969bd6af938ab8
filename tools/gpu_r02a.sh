#!/bin/bash
# round-2 evidence pass: new C3 headline bench, 2-rank self-spawn, ncu launch
# list + full capture, isolated-latency sweeps of the row template
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --gpus 2 --steps 64 --warmup 8 --no-subgraphs --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-subgraphs > gpurun_out/bench_under_ncu.log 2>&1
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prof -f \
    python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
for g in ln_4096x768 bert_resln bert_cut; do
  timeout 600 python tools/sweep_env.py $g 'STITCH_ROW_PIPE=1,2' 'STITCH_ROW_BLOCK=0,128,256,512' >> gpurun_out/sweep_rows.jsonl 2>&1
done
echo done
