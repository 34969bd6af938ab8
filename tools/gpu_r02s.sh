#!/bin/bash
# evidence pass 2 (round 2 final code): GPU suite, smoke, bench + reference arm, launch list, ncu headline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-subgraphs > gpurun_out/bench_under_ncu.log 2>&1
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prof -f \
    python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
echo done
