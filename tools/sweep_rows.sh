for gname in ln_4096x768 bert_resln attn_softmax ln2pass_4096x768; do
python tools/sweep_env.py $gname "STITCH_ROW_BLOCK=-1,64,128,256,512,1024" 2>&1
done
python tools/sweep_env.py ln_4096x768 "STITCH_ROW_BLOCK=-1,256 STITCH_ROW_NJ=6,12,24" 2>&1
