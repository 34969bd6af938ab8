import os,sys; sys.path.insert(0,'.')
import torch
from paper_2009_10924_b200 import stitch, shard
text=open('paper_2009_10924_b200/graphs/attn_softmax.graph').read()
g=stitch.Graph(text); inputs=stitch.random_inputs(g,1)
pin_in = {t.name: torch.from_numpy(inputs[t.name]).pin_memory().numpy() for t in g.params}
pin_out = {t.name: torch.empty(t.dims, dtype=torch.float32).pin_memory().numpy() for t in g.outputs}
for n in (4,8):
    cx=stitch.ChunkedExecutor(text, shard.RULES['attn_softmax'], n)
    cx.run(pin_in,out=pin_out); cx.run(pin_in,out=pin_out)
    os.environ['STITCH_CHUNK_TRACE']='1'
    cx.run(pin_in,out=pin_out)
    os.environ['STITCH_CHUNK_TRACE']='0'
