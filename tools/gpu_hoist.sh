python -m pytest tests/test_gpu_exec.py -x -q 2>&1 | tail -2
for g in ln_4096x768 ln2pass_4096x768 bert_resln attn_softmax bert_gelu colreduce dien_T10 bert_cut; do python tools/sweep_env.py $g "STITCH_PDL_HOIST=0,1" | cut -c1-160; done
python tools/calibrate_b200.py --out gpurun_out/b200.cfg --json gpurun_out/calibration_b200.json > gpurun_out/calib.log 2>&1; grep shuffle gpurun_out/b200.cfg
