"""Generators for the composite config graphs.

    python -m paper_2009_10924_b200.graphs.make_graphs      # rewrites *.graph here

bert_layer.graph   A.4: FFN GEMMs as opaque_compute + bias/GELU + bias/residual/LN
bert_cut.graph     A.4-cut: GEMM outputs promoted to parameters, outputs gl and y
dien_T<T>.graph    A.5: DIEN AUGRU recurrence, T steps, batch 256, hidden 36, with the
                   attention softmax over the time axis feeding every step
dien_cut_T<T>.graph  A.5 with every opaque GEMM output promoted to a parameter
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def _read(name):
    with open(os.path.join(HERE, name)) as f:
        return [l for l in f.read().splitlines() if l and not l.startswith("#")]


def bert(cut):
    gelu = [l for l in _read("bert_gelu.graph") if not l.startswith("output")]
    resln = [l for l in _read("bert_resln.graph")]
    out = ["# BERT-base FFN memory-intensive subgraphs, tokens 4096 (SURVEY.md Appendix A.4%s)"
           % ("-cut" if cut else "")]
    out.append("h = parameter : f32[4096,768]")
    if cut:
        out += gelu
    else:
        out.append("w1 = parameter : f32[768,3072]")
        out.append("b1 = parameter : f32[3072]")
        out.append("ffn1 = opaque_compute(h, w1) : f32[4096,3072]")
        out += [l for l in gelu if not l.startswith(("ffn1 =", "b1 ="))]
        out.append("w2 = parameter : f32[3072,768]")
    for l in resln:
        if l.startswith("h = "):
            continue
        if l.startswith("ffn2 = ") and not cut:
            l = "ffn2 = opaque_compute(gl, w2) : f32[4096,768]"
        out.append(l)
    if cut:
        out.append("output gl")
    return "\n".join(out) + "\n"


def dien(T, cut, B=256, H=36):
    L = ["# DIEN-style AUGRU recurrence, T=%d, batch %d, hidden %d (SURVEY.md Appendix A.5%s)"
         % (T, B, H, ", opaque outputs as parameters" if cut else "")]
    S = "f32[%d,%d]" % (B, H)
    L += ["h0 = parameter : %s" % S,
          "bu = parameter : f32[%d]" % H, "br = parameter : f32[%d]" % H,
          "bh = parameter : f32[%d]" % H,
          "bub = broadcast(bu) dims=[1] : %s" % S, "brb = broadcast(br) dims=[1] : %s" % S,
          "bhb = broadcast(bh) dims=[1] : %s" % S,
          "c0 = constant value=0 : f32[]", "c1 = constant value=1 : f32[]",
          "c0b = broadcast(c0) : %s" % S, "c1b = broadcast(c1) : %s" % S]
    # DIEN's attention: one score per (sequence, step) from the attention MLP
    # over every interest state and the target ad (opaque GEMMs), softmax over
    # the time axis (reduce_max / reduce_sum over T).  The IR has no reshape,
    # so step t's weight column [B,1] is squeezed to [B] by a reduce_sum over
    # its size-1 axis (exact: one term).
    if cut:
        L += ["sc = parameter : f32[%d,%d]" % (B, T)]
    else:
        L += ["x%d = parameter : %s" % (t, S) for t in range(T)]
        L += ["tgt = parameter : %s" % S,
              "sc = opaque_compute(%s, tgt) : f32[%d,%d]" % (", ".join("x%d" % t for t in range(T)), B, T)]
    L += ["scm = reduce_max(sc) axes=1 : f32[%d]" % B,
          "scmb = broadcast(scm) dims=[0] : f32[%d,%d]" % (B, T),
          "scs = sub(sc, scmb)", "sce = exp(scs)",
          "scz = reduce_sum(sce) axes=1 : f32[%d]" % B,
          "sczb = broadcast(scz) dims=[0] : f32[%d,%d]" % (B, T),
          "att = div(sce, sczb)"]
    h = "h0"
    for t in range(T):
        if cut:
            L += ["zu%d = parameter : %s" % (t, S), "zr%d = parameter : %s" % (t, S),
                  "uh%d = parameter : %s" % (t, S), "xh%d = parameter : %s" % (t, S)]
        else:
            L += ["zu%d = opaque_compute(x%d, %s) : %s" % (t, t, h, S),
                  "zr%d = opaque_compute(x%d, %s) : %s" % (t, t, h, S),
                  "uh%d = opaque_compute(%s) : %s" % (t, h, S),
                  "xh%d = opaque_compute(x%d) : %s" % (t, t, S)]
        for g, b in (("u", "bub"), ("r", "brb")):
            L += ["%sa%d = add(z%s%d, %s)" % (g, t, g, t, b),
                  "%sn%d = sub(c0b, %sa%d)" % (g, t, g, t),
                  "%se%d = exp(%sn%d)" % (g, t, g, t),
                  "%sd%d = add(c1b, %se%d)" % (g, t, g, t),
                  "%s%d = div(c1b, %sd%d)" % (g, t, g, t)]
        L += ["rh%d = mul(r%d, uh%d)" % (t, t, t),
              "hx%d = add(xh%d, rh%d)" % (t, t, t),
              "hb%d = add(hx%d, bhb)" % (t, t),
              "hc%d = tanh(hb%d)" % (t, t),
              "ats%d = slice(att) starts=[0,%d] limits=[%d,%d]" % (t, t, B, t + 1),
              "att%d = reduce_sum(ats%d) axes=1 : f32[%d]" % (t, t, B),
              "attb%d = broadcast(att%d) dims=[0] : %s" % (t, t, S),
              "au%d = mul(attb%d, u%d)" % (t, t, t),
              "om%d = sub(c1b, au%d)" % (t, t),
              "keep%d = mul(om%d, %s)" % (t, t, h),
              "upd%d = mul(au%d, hc%d)" % (t, t, t),
              "h%d = add(keep%d, upd%d)" % (t + 1, t, t)]
        h = "h%d" % (t + 1)
    L.append("output %s" % h)
    return "\n".join(L) + "\n"


def main():
    files = {"bert_layer.graph": bert(False), "bert_cut.graph": bert(True)}
    for T in (10, 20):
        files["dien_T%d.graph" % T] = dien(T, False)
        files["dien_cut_T%d.graph" % T] = dien(T, True)
    for name, text in files.items():
        with open(os.path.join(HERE, name), "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
