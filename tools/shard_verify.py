"""Multi-GPU verification of independent batch shards.

    torchrun --nproc-per-node N tools/shard_verify.py [graph]

Each rank plans ITS shard graph (shapes change -> plans are recomputed per
shard), executes it as stitched sm_100a kernels in one CUDA Graph on its own
GPU with its slice of the full-graph inputs, times it (no collective on the
data path), then -- outside the timed region -- NCCL all_gather brings the
shard outputs to rank 0, which checks them against the oracle evaluation of
the FULL graph.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from oracle import numpy_oracle as no
    from paper_2009_10924_b200 import stitch
    from paper_2009_10924_b200.shard import RULES

    name = sys.argv[1] if len(sys.argv) > 1 else "attn_softmax"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rule = RULES[name]
    with open(os.path.join(stitch.GRAPHS, name + ".graph")) as f:
        text = f.read()
    g_full = no.parse_graph(text)
    full_inputs = no.random_inputs(g_full, 1)
    g = stitch.Graph(rule.graph_text(text, world))
    ex = stitch.Executor(stitch.Plan(g, "b200"), device=local)
    mine = rule.slice_inputs({k: v.astype(np.float32) for k, v in full_inputs.items()}, world, rank)
    ex.upload(mine)
    us, _ = ex.time(iters=100, warmup=10, sets=4)
    ex.launch()
    ex.sync()
    out = ex.download()
    gathered = {}
    for t in g.outputs:
        local_t = torch.from_numpy(out[t.name]).cuda()
        if world > 1:
            parts = [torch.empty_like(local_t) for _ in range(world)]
            dist.all_gather(parts, local_t)  # verification only, after timing
            gathered[t.name] = [p.cpu().numpy() for p in parts]
        else:
            gathered[t.name] = [out[t.name]]
    if rank == 0:
        got = rule.concat_outputs([{k: v[r] for k, v in gathered.items()} for r in range(world)])
        want = no.eval_reference(g_full, full_inputs)
        rep = stitch.compare(got, want, 1e-4, 1e-5)
        print(json.dumps({"graph": name, "ranks": world, "shard_us": round(us, 3), "pass": rep["pass"],
                          "max_abs": rep["max_abs"], "max_rel": rep["max_rel"]}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
