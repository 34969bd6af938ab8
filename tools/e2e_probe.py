"""e2e probe (diagnostics): host-buffer execution paths on one config graph:
plain (H2D all, graph, D2H all), pipelined chunks, zero-copy kernels."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2009_10924_b200 import stitch, shard

for name in sys.argv[1:] or ["attn_softmax", "ln_4096x768", "bert_gelu", "bert_resln"]:
    text = open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
    g = stitch.Graph(text)
    inputs = stitch.random_inputs(g, 1)
    pin_in = {t.name: torch.from_numpy(inputs[t.name]).pin_memory().numpy() for t in g.params}
    pin_out = {t.name: torch.empty(t.dims, dtype=torch.float32).pin_memory().numpy() for t in g.outputs}
    nbytes = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    ex = stitch.Executor(stitch.Plan(g, "b200"))
    ref = {k: v.copy() for k, v in ex.run(inputs).items()}

    def timed(fn, reps=20):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps

    rows = [("plain", lambda: ex.run(pin_in, out=pin_out))]
    full = shard.RULES[name].full
    shapes = {"chunked4": 4, "chunked8": 8}
    if full == 32:
        shapes.update({"taper_1_3_4x6_3_1": [1, 3, 4, 4, 4, 4, 4, 4, 3, 1], "taper_2_6x5_2": [2, 6, 6, 6, 6, 4, 2],
                       "taper_1_2_4x6_4_1": [1, 2, 4, 4, 4, 4, 4, 4, 4, 1]})
    else:
        u = full // 32
        shapes.update({"taper_1_3_4x6_3_1": [u * c for c in [1, 3, 4, 4, 4, 4, 4, 4, 3, 1]]})
    def d2h_copy(cx):
        def f():
            os.environ["STITCH_E2E_ZC_OUT"] = "0"
            try:
                cx.run(pin_in, out=pin_out)
            finally:
                os.environ.pop("STITCH_E2E_ZC_OUT", None)
        return f

    for label, ch in shapes.items():
        cx = stitch.ChunkedExecutor(text, shard.RULES[name], ch)
        rows.append((label, d2h_copy(cx)))
    rows.append(("zero_copy", lambda: ex.run_zero_copy(pin_in, pin_out)))
    for n in (2, 4, 8):
        cz = stitch.ChunkedExecutor(text, shard.RULES[name], n)

        rows.append(("chunked%d_zc_out" % n, lambda cz=cz: cz.run(pin_in, out=pin_out)))
    for label, fn in rows:
        s = timed(fn)
        same = all(np.array_equal(pin_out[k], ref[k]) for k in ref)
        print(json.dumps({"graph": name, "path": label, "us": round(s * 1e6, 1), "GBps": round(nbytes / s / 1e9, 2),
                          "bitwise_equal": same}), flush=True)
