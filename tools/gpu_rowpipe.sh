python -m pytest tests/test_gpu_exec.py -q -x 2>&1 | tail -1
for g in ln_4096x768 ln2pass_4096x768 bert_resln bert_cut attn_softmax; do python tools/sweep_env.py $g "STITCH_ROW_PIPE=1,2" | cut -c1-140; done
