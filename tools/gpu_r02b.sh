#!/bin/bash
# DIEN attention-score placeholder sizing + same-byte floors (events and ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dien or opaque or parity_mode or pack" > gpurun_out/pytest_dien.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dien.log
for g in dien_T10 dien_T20; do
  timeout 600 python tools/sweep_env.py $g 'STITCH_OPAQUE_CLUSTER=-1,1' >> gpurun_out/dien_sc_ab.jsonl 2>&1
done
timeout 600 python tools/floor_probe.py > gpurun_out/floor_probe.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/floor_ncu.csv python tools/floor_probe.py --ncu > gpurun_out/floor_ncu.log 2>&1
REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/config_ncu.csv python tools/ncu_target.py > gpurun_out/config_ncu.log 2>&1
echo done
