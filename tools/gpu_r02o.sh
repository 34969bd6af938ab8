#!/bin/bash
# ncu of the BERT-layer grid placeholders; 2-rank bench on one GPU (logic run)
mkdir -p gpurun_out
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn -c 2 -o gpurun_out/ffn -f \
    python tools/ncu_target.py bert_layer > gpurun_out/ncu_ffn.log 2>&1
timeout 900 python bench.py --gpus 2 --steps 256 --warmup 8 --no-cpu-baseline --no-subgraphs > gpurun_out/bench_2r.json 2> gpurun_out/bench_2r.err
echo done
