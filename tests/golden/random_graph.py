"""Restatement of the reference's test generator ``random_graph(seed, max_fusable)``
(/root/reference/proj/tests/test_util.hpp:16-30 SplitMix, 46-116 random_graph)
emitting graph TEXT in the reference format, so both planners can read the same
graph.  Graphs with an unused parameter (which parse_graph rejects as a dead
node) are returned as None."""

M64 = (1 << 64) - 1


class SplitMix:
    def __init__(self, seed):
        self.s = seed & M64

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def range(self, lo, hi):
        return lo + self.next() % (hi - lo + 1)


def random_graph_nodes(seed, max_fusable):
    rng = SplitMix(seed)
    rows = 4 << rng.range(0, 2)
    cols = 16 << rng.range(0, 2)
    full, red = [rows, cols], [rows]
    nodes = []  # (name, kind, operands, shape, attr)

    def add(name, kind, ops, shape, attr=""):
        nodes.append((name, kind, ops, shape, attr))
        return len(nodes) - 1

    full_pool, red_pool = [], []
    for i in range(rng.range(1, 2)):
        full_pool.append(add("p%d" % i, "parameter", [], full))
    nfuse = rng.range(3, max_fusable)
    i = 0
    while i < nfuse:
        name = "v%d" % i
        roll = rng.range(0, 9)
        if roll < 4 or (not red_pool and roll < 6):
            kind = ["add", "sub", "mul", "max"][rng.range(0, 3)]
            a = full_pool[rng.range(0, len(full_pool) - 1)]
            b = full_pool[rng.range(0, len(full_pool) - 1)]
            full_pool.append(add(name, kind, [a, b], full))
        elif roll < 6:
            a = red_pool[rng.range(0, len(red_pool) - 1)]
            b = red_pool[rng.range(0, len(red_pool) - 1)]
            red_pool.append(add(name, "add", [a, b], red))
        elif roll < 7:
            kind = "tanh" if rng.range(0, 1) else "exp"
            a = full_pool[rng.range(0, len(full_pool) - 1)]
            full_pool.append(add(name, kind, [a], full))
        elif roll < 9:
            kind = "reduce_sum" if rng.range(0, 1) else "reduce_max"
            a = full_pool[rng.range(0, len(full_pool) - 1)]
            red_pool.append(add(name, kind, [a], red, " axes=1"))
        elif red_pool:
            a = red_pool[rng.range(0, len(red_pool) - 1)]
            full_pool.append(add(name, "broadcast", [a], full, " dims=0"))
        else:
            continue
        i += 1
    consumed = {o for n in nodes for o in n[2]}
    outputs = [k for k, n in enumerate(nodes) if k not in consumed and n[1] != "parameter"]
    if not outputs:
        outputs = [len(nodes) - 1]
    return nodes, outputs


def random_graph_text(seed, max_fusable=10):
    nodes, outputs = random_graph_nodes(seed, max_fusable)
    consumed = {o for n in nodes for o in n[2]}
    if any(n[1] == "parameter" and k not in consumed for k, n in enumerate(nodes)):
        return None
    lines = []
    for name, kind, ops, shape, attr in nodes:
        lines.append("%s = %s(%s)%s : f32[%s]" % (name, kind, ", ".join(nodes[o][0] for o in ops),
                                                 attr, ",".join(str(d) for d in shape)))
    lines += ["output " + nodes[o][0] for o in outputs]
    return "\n".join(lines) + "\n"
