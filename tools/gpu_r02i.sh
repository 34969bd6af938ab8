#!/bin/bash
# evidence pass after the row fixes: bench (serial + one-call + call floor), ncu full captures of the configs
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "bert_cut or heterogeneous or packing" > gpurun_out/pytest_cut.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cut.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-subgraphs > gpurun_out/bench_under_ncu.log 2>&1
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prof -f \
    python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
echo done
