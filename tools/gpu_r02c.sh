#!/bin/bash
# bert_cut body order / interleave A/B; DIEN in-graph timeline + lane map
mkdir -p gpurun_out
timeout 600 python tools/sweep_env.py bert_cut 'STITCH_BODY_ORDER=0,1' 'STITCH_INTERLEAVE=0,1' > gpurun_out/bert_cut_order_ab.jsonl 2>&1
timeout 300 python tools/trace_timeline.py dien_T10 > gpurun_out/dien_timeline.txt 2>&1
STITCH_LANES=1 timeout 300 python -c "
import os,sys; sys.path.insert(0,'.')
from paper_2009_10924_b200 import stitch
g=stitch.Graph.from_file(os.path.join(stitch.GRAPHS,'dien_T10.graph'))
ex=stitch.Executor(stitch.Plan(g,'b200')); ex.upload(stitch.random_inputs(g,1)); ex.time(iters=5,warmup=1)
" > gpurun_out/dien_lanes.txt 2>&1
echo done
