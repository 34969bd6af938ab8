"""Does the operand layout of B matter for the TF32 tcgen05 GEMM?  Times the
CUTLASS configurations of csrc/kernels/gemm_sm100.cu directly (the C++
entry point stitch::gpu::gemm_tf32 in libstitch_b200.so) on BERT's two FFN
shapes: B row-major [K,N] (variants 0 / 3, what the executor runs) vs B
column-major, i.e. B^T stored [N,K] (K-major; variants 7 / 6).  CUDA events
on the launching stream, best of 20 after warm-up, plus a max-abs check of
the two layouts against each other."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

lib = stitch.lib()
fn = getattr(lib, "_ZN6stitch3gpu9gemm_tf32EibPKfS2_S2_PfiiiPvmP11CUstream_st")
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_int, ctypes.c_bool] + [ctypes.c_void_p] * 4 + [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_size_t,
                                                                                         ctypes.c_void_p]
ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()


def run(v, fused, A, B, bias, D, M, N, K):
    rc = fn(v, fused, A.data_ptr(), B.data_ptr(), bias.data_ptr() if fused else None, D.data_ptr(), M, N, K,
            ws.data_ptr(), ws.numel(), stream.cuda_stream)
    if rc:
        raise RuntimeError("variant %d rc %d" % (v, rc))


def time_us(f, reps=20):
    for _ in range(3):
        f()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f()
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best


torch.manual_seed(0)
for name, M, N, K, fused, (vr, vc) in [("ffn2", 4096, 768, 3072, False, (3, 6)), ("ffn1", 4096, 3072, 768, True, (0, 7)),
                                       ("ffn2_256", 4096, 768, 3072, False, (0, 7))]:
    A = torch.rand(M, K, device="cuda") * 2 - 1
    B = torch.rand(K, N, device="cuda") * 2 - 1
    Bt = B.t().contiguous()
    bias = torch.rand(N, device="cuda")
    D1 = torch.empty(M, N, device="cuda")
    D2 = torch.empty(M, N, device="cuda")
    t_row = time_us(lambda: run(vr, fused, A, B, bias, D1, M, N, K))
    t_col = time_us(lambda: run(vc, fused, A, Bt, bias, D2, M, N, K))
    torch.cuda.synchronize()
    fl = 2 * M * N * K
    print(json.dumps({"gemm": name, "mnk": [M, N, K], "fused_bias_gelu": fused, "variant_row_major_B": vr,
                      "us_row_major_B": round(t_row, 2), "tflops_row": round(fl / t_row / 1e6, 1),
                      "variant_col_major_B": vc, "us_col_major_B": round(t_col, 2), "tflops_col": round(fl / t_col / 1e6, 1),
                      "max_abs_diff": float((D1 - D2).abs().max())}), flush=True)
