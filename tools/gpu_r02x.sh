#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "resident or dien" > gpurun_out/pytest_x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_x.log
for gname in dien_T10 dien_T20; do timeout 600 python tools/sweep_env.py $gname 'STITCH_RESIDENT_HANDOFF=0,1' >> gpurun_out/resident_handoff.jsonl 2>&1; done
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_exec.py -q -x -k "resident_template_matches" > gpurun_out/racecheck_handoff.log 2>&1
tail -n 2 gpurun_out/racecheck_handoff.log
echo done
