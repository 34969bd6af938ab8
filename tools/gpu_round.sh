#!/bin/bash
# One gpurun evidence pass: gpu tests, smoke, bench (+ clocks), ncu launch list
# of the bench, one ncu --set full capture per config kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ "${NCU:-1}" = "1" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -s 0 -c 40 -o gpurun_out/prof -f \
    python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
fi
echo done
