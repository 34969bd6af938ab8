for gname in ln_4096x768 bert_resln attn_softmax bert_gelu colreduce; do
python tools/sweep_env.py $gname "STITCH_NVRTC_DEFINES=none,STITCH_L2_256B,STITCH_ST_CS,STITCH_L2_256B:STITCH_ST_CS" 2>&1
done
