// Model mode (non-parity): a matmul-shaped opaque_compute
// followed by the plan's bias + GELU(tanh) pattern runs as ONE sm_100a kernel:
// a CUTLASS 4.x TF32 tcgen05 GEMM (2-SM 256x256x32 tiles, TMA operand
// loads, TMEM accumulators) whose epilogue adds the per-column bias and
// applies GELU(tanh) --
// the [M,N] GEMM output never reaches HBM.  Instantiated here from the CUTLASS
// headers vendored in the image (flashinfer/data/cutlass); without them the
// entry point reports "unavailable" and the executor keeps cuBLASLt + the
// stitched kernel.
// griddepcontrol in the CUTLASS kernels: the TMA load, bias load and tile
// scheduler warps wait on the producer grid before touching global memory,
// so the GEMM may be launched with programmatic dependent launch
// (gemm_tf32_launch(pdl = true)); without this define those waits compile
// to nothing and a PDL launch would race its producer
#define CUTLASS_ENABLE_GDC_FOR_SM100 1
#include <cstddef>
#include <type_traits>
#include <cuda_runtime.h>

#if __has_include("cutlass/cutlass.h")
#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/thread/activation.h"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"
#define STC_HAVE_CUTLASS 1
#endif

namespace stitch::gpu {

#ifdef STC_HAVE_CUTLASS
namespace {
using namespace cute;

// GELU(tanh) epilogue: CUTLASS's GELU_taylor, 0.5 z (1 + tanh(z (k0 + k1 z^2)))
// with tanh.approx.f32 (MUFU.TANH, rel err ~5e-4).  An accurate tanhf (the
// graph's own op order) in the epilogue made the kernel 56.5 vs 38.3 us cold
// for [4096x768]x[768x3072] (profiles/r02/gemm/fused_gemm_variants.txt): the
// epilogue warps are few and the accurate tanh sequence long.  TF32 operand
// rounding (~1e-3 relative) dominates the error either way.
using Row = cutlass::layout::RowMajor;
using GeluFusion =
    cutlass::epilogue::fusion::LinCombPerColBiasEltAct<cutlass::epilogue::thread::GELU_taylor, float, float, float>;
using PlainFusion = cutlass::epilogue::fusion::LinearCombination<float, float, float, float>;

// one TF32 tcgen05 GEMM configuration: MMA tile, cluster (2 along M = the
// 2-SM cta_group::2 MMA), tile scheduler (void = data-parallel persistent),
// epilogue fusion
template <class MmaTile, class Cluster, class Sched, class Fusion, class LayoutB = Row>
struct Cfg {
  using Epilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTile, Cluster,
      cutlass::epilogue::collective::EpilogueTileAuto, float, float, float, Row, 4, float, Row, 4,
      cutlass::epilogue::collective::EpilogueScheduleAuto, Fusion>::CollectiveOp;
  using Mainloop = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, Row, 4, float, LayoutB, 4, float, MmaTile, Cluster,
      cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epilogue::SharedStorage))>,
      cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
  using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Mainloop, Epilogue, Sched>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;
  static constexpr bool kFused = !std::is_same_v<Fusion, PlainFusion>;

  static typename Gemm::Arguments args(const float* A, const float* B, const float* bias, float* D, int M, int N, int K) {
    auto sA = cutlass::make_cute_packed_stride(typename Kernel::StrideA{}, cute::make_shape(M, K, 1));
    auto sB = cutlass::make_cute_packed_stride(typename Kernel::StrideB{}, cute::make_shape(N, K, 1));
    auto sC = cutlass::make_cute_packed_stride(typename Kernel::StrideC{}, cute::make_shape(M, N, 1));
    auto sD = cutlass::make_cute_packed_stride(typename Kernel::StrideD{}, cute::make_shape(M, N, 1));
    typename Gemm::Arguments a{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, 1}, {A, sA, B, sB},
                               {{}, nullptr, sC, D, sD}};
    a.epilogue.thread.alpha = 1.f;
    a.epilogue.thread.beta = 0.f;
    if constexpr (kFused) a.epilogue.thread.bias_ptr = bias;
    return a;
  }
  static long long workspace(int M, int N, int K) {
    auto a = args(nullptr, nullptr, nullptr, nullptr, M, N, K);
    if (Gemm::can_implement(a) != cutlass::Status::kSuccess) return -1;
    return static_cast<long long>(Gemm::get_workspace_size(a));
  }
  static int run(const float* A, const float* B, const float* bias, float* D, int M, int N, int K, void* ws,
                 size_t ws_bytes, cudaStream_t stream, bool pdl) {
    auto a = args(A, B, bias, D, M, N, K);
    Gemm gemm;
    if (Gemm::get_workspace_size(a) > ws_bytes || gemm.can_implement(a) != cutlass::Status::kSuccess) return 1;
    if (gemm.initialize(a, ws, stream) != cutlass::Status::kSuccess) return 2;
    return gemm.run(stream, nullptr, pdl) == cutlass::Status::kSuccess ? 0 : 2;
  }
};

using T256x256 = Shape<_256, _256, _32>;
using T256x192 = Shape<_256, _192, _32>;
using T128x192 = Shape<_128, _192, _32>;

using C2 = Shape<_2, _1, _1>;
using C22 = Shape<_2, _2, _1>;  // 2 SM pairs along N: A tiles multicast by TMA
using C1 = Shape<_1, _1, _1>;
using SK = cutlass::gemm::StreamKScheduler;
using Col = cutlass::layout::ColumnMajor;

// variants (ids are the STITCH_GEMM_PLAIN / STITCH_GEMM_FUSED values):
//   0  2-SM 256x256 data-parallel (fused default; plain default is cuBLASLt)
//   1  2-SM 256x256 stream-K: BERT's ffn2 ([4096,3072] x [3072,768]) has
//      only 48 output tiles of 256x256 for 74 SM pairs
//   2  1-SM 128x192 data-parallel: 128 ffn2 tiles for 148 SMs, one wave
//   3  2-SM 256x192 data-parallel
//   4  2-SM 256x256, clusters of 2 pairs along N (A multicast)
//   5  2-SM 256x192, clusters of 2 pairs along N (A multicast)
//   6  2-SM 256x192 with B column-major (K-major: B^T stored [N,K]) -- layout
//      probe only (tools/gemm_layout_probe.py); the executor's weights are
//      row-major [K,N] and it never selects 6 / 7
//   7  2-SM 256x256 with B column-major (probe only)
// (64-deep K tiles, 2-SM 256x256 / 256x192, measured 13-45% slower: fewer
// pipeline stages fit; profiles/r02/gemm/gemm_variants_k64.jsonl)
template <class Fusion>
long long ws_of(int v, int M, int N, int K) {
  switch (v) {
    case 0: return Cfg<T256x256, C2, void, Fusion>::workspace(M, N, K);
    case 1: return Cfg<T256x256, C2, SK, Fusion>::workspace(M, N, K);
    case 2: return Cfg<T128x192, C1, void, Fusion>::workspace(M, N, K);
    case 3: return Cfg<T256x192, C2, void, Fusion>::workspace(M, N, K);
    case 4: return Cfg<T256x256, C22, void, Fusion>::workspace(M, N, K);
    case 5: return Cfg<T256x192, C22, void, Fusion>::workspace(M, N, K);
    case 6: return Cfg<T256x192, C2, void, Fusion, Col>::workspace(M, N, K);
    case 7: return Cfg<T256x256, C2, void, Fusion, Col>::workspace(M, N, K);
    default: return -1;
  }
}
template <class Fusion>
int run_of(int v, const float* A, const float* B, const float* bias, float* D, int M, int N, int K, void* ws, size_t wsb,
           cudaStream_t s, bool pdl) {
  switch (v) {
    case 0: return Cfg<T256x256, C2, void, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 1: return Cfg<T256x256, C2, SK, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 2: return Cfg<T128x192, C1, void, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 3: return Cfg<T256x192, C2, void, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 4: return Cfg<T256x256, C22, void, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 5: return Cfg<T256x192, C22, void, Fusion>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 6: return Cfg<T256x192, C2, void, Fusion, Col>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    case 7: return Cfg<T256x256, C2, void, Fusion, Col>::run(A, B, bias, D, M, N, K, ws, wsb, s, pdl);
    default: return 1;
  }
}
}  // namespace
#endif

// D[M,N] = A[M,K] . B[K,N] (+ per-column bias, then GELU(tanh), when `fused`),
// row-major f32, TF32 tensor cores, CUTLASS configuration `variant` (above).
// 0 = launched on `stream`; 1 = unavailable (no CUTLASS / shape not
// implementable / unknown variant); 2 = launch error.  The workspace must
// hold gemm_tf32_workspace() bytes and belong to this GEMM (stream-K keeps
// its fix-up partials and flags there).
// pdl: launched with programmatic stream serialization (the kernel's
// griddepcontrol.wait orders it after its producer)
int gemm_tf32_launch(int variant, bool fused, bool pdl, const float* A, const float* B, const float* bias, float* D, int M,
                     int N, int K, void* workspace, size_t workspace_bytes, cudaStream_t stream) {
#ifdef STC_HAVE_CUTLASS
  return fused ? run_of<GeluFusion>(variant, A, B, bias, D, M, N, K, workspace, workspace_bytes, stream, pdl)
               : run_of<PlainFusion>(variant, A, B, bias, D, M, N, K, workspace, workspace_bytes, stream, pdl);
#else
  (void)variant, (void)fused, (void)pdl, (void)A, (void)B, (void)bias, (void)D, (void)M, (void)N, (void)K,
      (void)workspace, (void)workspace_bytes, (void)stream;
  return 1;
#endif
}

int gemm_tf32(int variant, bool fused, const float* A, const float* B, const float* bias, float* D, int M, int N, int K,
              void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  return gemm_tf32_launch(variant, fused, false, A, B, bias, D, M, N, K, workspace, workspace_bytes, stream);
}

// workspace bytes of that configuration for this shape; -1 = not implementable
long long gemm_tf32_workspace(int variant, bool fused, int M, int N, int K) {
#ifdef STC_HAVE_CUTLASS
  return fused ? ws_of<GeluFusion>(variant, M, N, K) : ws_of<PlainFusion>(variant, M, N, K);
#else
  (void)variant, (void)fused, (void)M, (void)N, (void)K;
  return -1;
#endif
}

// D[M,N] = GELU(A[M,K] . B[K,N] + bias[N]) on the default fused configuration
int gemm_bias_gelu_tf32(const float* A, const float* B, const float* bias, float* D, int M, int N, int K, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream) {
  return gemm_tf32(0, true, A, B, bias, D, M, N, K, workspace, workspace_bytes, stream);
}

// whether the fused path can run this shape (host-side check, no launch)
bool gemm_bias_gelu_supported(int M, int N, int K, size_t workspace_bytes) {
  const long long ws = gemm_tf32_workspace(0, true, M, N, K);
  return ws >= 0 && static_cast<size_t>(ws) <= workspace_bytes;
}

}  // namespace stitch::gpu
