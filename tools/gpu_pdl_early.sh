python tools/calibrate_b200.py --out gpurun_out/b200.cfg --json gpurun_out/calibration_b200.json > gpurun_out/calib.log 2>&1
for g in ln_4096x768 bert_resln attn_softmax dien_T10; do python tools/sweep_env.py $g "STITCH_PDL_EARLY=0,1" | cut -c1-200; done
