python -m pytest tests/test_gpu_exec.py -q -k "edge_shapes" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
cat > /tmp/g1.graph <<'G'
x = parameter : f32[8,65536]
m = reduce_max(x) axes=1
mb = broadcast(m) dims=0 : f32[8,65536]
sh = sub(x, mb)
e = exp(sh)
s = reduce_sum(e) axes=1
sb = broadcast(s) dims=0 : f32[8,65536]
y = div(e, sb)
output y
G
python - <<'P'
import sys, os, math; sys.path.insert(0,'.')
from paper_2009_10924_b200 import stitch
for cl in ("1","0"):
    os.environ["STITCH_ROW_CLUSTER"]=cl
    for rows, cols in [(8,65536),(16,8192),(4,262144)]:
        txt=open('/tmp/g1.graph').read().replace('[8,65536]','[%d,%d]'%(rows,cols))
        g=stitch.Graph(txt); ex=stitch.Executor(stitch.Plan(g,'b200')); ex.upload(stitch.random_inputs(g,1))
        d=ex.describe(); per=sum(t.nbytes for t in g.params)+sum(t.nbytes for t in g.outputs)
        us=ex.time_batched(steps=64,warmup=8,sets=min(64,max(2,math.ceil(8*126*2**20/per))),steps_per_graph=8)
        print("cluster" if cl=="1" else "no-cluster", rows, cols, [(k['template'],k['grid'],k['block']) for k in d], round(us,2), "us", round(sum(k['bytes'] for k in d)/us/1e3,1), "GB/s")
P
