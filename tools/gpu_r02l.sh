#!/bin/bash
# resident cluster size + step timeline; TMA vs register LN under ncu
mkdir -p gpurun_out
timeout 300 python tools/resident_timeline.py dien_T10 > gpurun_out/resident_timeline_c16.txt 2>&1
STITCH_RESIDENT_CLUSTER=8 timeout 300 python tools/resident_timeline.py dien_T10 > gpurun_out/resident_timeline_c8.txt 2>&1
for gname in dien_T10 dien_T20; do
  timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_CLUSTER=8,16' >> gpurun_out/resident_cluster.jsonl 2>&1
done
REPS=2 timeout 600 ncu --set full --clock-control none -k regex:k0_cnb -c 2 -o gpurun_out/ln_reg -f python tools/ncu_target.py ln_4096x768 > gpurun_out/ncu_ln.log 2>&1
STITCH_STAGE=1 STITCH_STAGES=4 REPS=2 timeout 600 ncu --set full --clock-control none -k regex:k0_cnb -c 2 -o gpurun_out/ln_tma -f python tools/ncu_target.py ln_4096x768 >> gpurun_out/ncu_ln.log 2>&1
echo done
