// Model mode (non-parity): a matmul-shaped opaque_compute
// followed by the plan's bias + GELU(tanh) pattern runs as ONE sm_100a kernel:
// a CUTLASS 4.x TF32 tcgen05 GEMM (2-SM 256x256x32 tiles, TMA operand
// loads, TMEM accumulators) whose epilogue adds the per-column bias and
// applies GELU(tanh) --
// the [M,N] GEMM output never reaches HBM.  Instantiated here from the CUTLASS
// headers vendored in the image (flashinfer/data/cutlass); without them the
// entry point reports "unavailable" and the executor keeps cuBLASLt + the
// stitched kernel.
#include <cstddef>
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
using MmaTile = Shape<_256, _256, _32>;
using Cluster = Shape<_2, _1, _1>;
using Fusion = cutlass::epilogue::fusion::LinCombPerColBiasEltAct<cutlass::epilogue::thread::GELU_taylor, float, float, float>;
using Epilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTile, Cluster, cutlass::epilogue::collective::EpilogueTileAuto,
    float, float, float, Row, 4, float, Row, 4, cutlass::epilogue::collective::EpilogueScheduleAuto, Fusion>::CollectiveOp;
using Mainloop = typename cutlass::gemm::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, Row, 4, float, Row, 4, float, MmaTile, Cluster,
    cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epilogue::SharedStorage))>,
    cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Mainloop, Epilogue>;
using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;
// the same fused kernel on the stream-K tile scheduler: ffn1 ([4096,768] x
// [768,3072]) is 192 tiles of 256x256 for 74 SM pairs, 2.6 waves
using KernelSk =
    cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Mainloop, Epilogue, cutlass::gemm::StreamKScheduler>;
using GemmSkFused = cutlass::gemm::device::GemmUniversalAdapter<KernelSk>;

template <class G>
typename G::Arguments make_args_t(const float* A, const float* B, const float* bias, float* D, int M, int N, int K) {
  using Kn = typename G::GemmKernel;
  auto sA = cutlass::make_cute_packed_stride(typename Kn::StrideA{}, cute::make_shape(M, K, 1));
  auto sB = cutlass::make_cute_packed_stride(typename Kn::StrideB{}, cute::make_shape(N, K, 1));
  auto sC = cutlass::make_cute_packed_stride(typename Kn::StrideC{}, cute::make_shape(M, N, 1));
  auto sD = cutlass::make_cute_packed_stride(typename Kn::StrideD{}, cute::make_shape(M, N, 1));
  typename G::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, 1}, {A, sA, B, sB},
                             {{}, nullptr, sC, D, sD}};
  args.epilogue.thread.alpha = 1.f;
  args.epilogue.thread.beta = 0.f;
  args.epilogue.thread.bias_ptr = bias;
  return args;
}
typename Gemm::Arguments make_args(const float* A, const float* B, const float* bias, float* D, int M, int N, int K) {
  return make_args_t<Gemm>(A, B, bias, D, M, N, K);
}

// Plain D = A . B for the GEMMs with no fused epilogue, on CUTLASS's stream-K
// tile scheduler.  BERT's ffn2 ([4096,3072] x [3072,768]) has only 16 x 3 =
// 48 output tiles of 256x256 for 74 SM pairs: a data-parallel grid leaves a
// third of the pairs idle, stream-K splits the K loop of the remainder over
// them (deterministic fix-up in the workspace).
using SkFusion = cutlass::epilogue::fusion::LinearCombination<float, float, float, float>;
using SkEpilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTile, Cluster, cutlass::epilogue::collective::EpilogueTileAuto,
    float, float, float, Row, 4, float, Row, 4, cutlass::epilogue::collective::EpilogueScheduleAuto, SkFusion>::CollectiveOp;
using SkMainloop = typename cutlass::gemm::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, float, Row, 4, float, Row, 4, float, MmaTile, Cluster,
    cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename SkEpilogue::SharedStorage))>,
    cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;
using SkKernel =
    cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, SkMainloop, SkEpilogue, cutlass::gemm::StreamKScheduler>;
using SkGemm = cutlass::gemm::device::GemmUniversalAdapter<SkKernel>;

// splits > 1: split-K with that many splits; 0: CUTLASS's stream-K heuristic
typename SkGemm::Arguments make_sk_args(const float* A, const float* B, float* D, int M, int N, int K, int splits) {
  auto sA = cutlass::make_cute_packed_stride(typename SkKernel::StrideA{}, cute::make_shape(M, K, 1));
  auto sB = cutlass::make_cute_packed_stride(typename SkKernel::StrideB{}, cute::make_shape(N, K, 1));
  auto sC = cutlass::make_cute_packed_stride(typename SkKernel::StrideC{}, cute::make_shape(M, N, 1));
  auto sD = cutlass::make_cute_packed_stride(typename SkKernel::StrideD{}, cute::make_shape(M, N, 1));
  typename SkGemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, 1}, {A, sA, B, sB},
                                  {{}, nullptr, sC, D, sD}};
  args.epilogue.thread.alpha = 1.f;
  args.epilogue.thread.beta = 0.f;
  if (splits > 1) args.scheduler.splits = splits;
  return args;
}
}  // namespace
#endif

// D[M,N] = A[M,K] . B[K,N], row-major f32, TF32 tensor cores, stream-K
// (splits > 1: split-K).  Same return codes as gemm_bias_gelu_tf32.  The
// workspace must hold gemm_tf32_streamk_workspace() bytes and belong to this
// GEMM alone (it carries the fix-up partials and their flags).
int gemm_tf32_streamk(const float* A, const float* B, float* D, int M, int N, int K, int splits, void* workspace,
                      size_t workspace_bytes, cudaStream_t stream) {
#ifdef STC_HAVE_CUTLASS
  auto args = make_sk_args(A, B, D, M, N, K, splits);
  SkGemm gemm;
  if (SkGemm::get_workspace_size(args) > workspace_bytes || gemm.can_implement(args) != cutlass::Status::kSuccess) return 1;
  if (gemm.initialize(args, workspace, stream) != cutlass::Status::kSuccess) return 2;
  return gemm.run(stream) == cutlass::Status::kSuccess ? 0 : 2;
#else
  (void)A, (void)B, (void)D, (void)M, (void)N, (void)K, (void)splits, (void)workspace, (void)workspace_bytes, (void)stream;
  return 1;
#endif
}

// workspace bytes the stream-K GEMM needs for this shape; -1 = not
// implementable.  Split-K (splits > 1) is refused: its launch could not be
// captured into the plan's CUDA graph ("stream capture of the plan failed")
long long gemm_tf32_streamk_workspace(int M, int N, int K, int splits) {
  if (splits > 1) return -1;
#ifdef STC_HAVE_CUTLASS
  auto args = make_sk_args(nullptr, nullptr, nullptr, M, N, K, splits);
  if (SkGemm::can_implement(args) != cutlass::Status::kSuccess) return -1;
  return static_cast<long long>(SkGemm::get_workspace_size(args));
#else
  (void)M, (void)N, (void)K, (void)splits;
  return -1;
#endif
}

// D[M,N] = GELU(A[M,K] . B[K,N] + bias[N]), all row-major f32, TF32 tensor
// cores.  0 = launched on `stream`; 1 = unavailable (no CUTLASS / shape not
// implementable); 2 = launch error.
int gemm_bias_gelu_tf32(const float* A, const float* B, const float* bias, float* D, int M, int N, int K, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream) {
#ifdef STC_HAVE_CUTLASS
  auto args = make_args(A, B, bias, D, M, N, K);
  Gemm gemm;
  if (Gemm::get_workspace_size(args) > workspace_bytes || gemm.can_implement(args) != cutlass::Status::kSuccess) return 1;
  if (gemm.initialize(args, workspace, stream) != cutlass::Status::kSuccess) return 2;
  return gemm.run(stream) == cutlass::Status::kSuccess ? 0 : 2;
#else
  (void)A, (void)B, (void)bias, (void)D, (void)M, (void)N, (void)K, (void)workspace, (void)workspace_bytes, (void)stream;
  return 1;
#endif
}

// the fused GEMM on the stream-K scheduler; the workspace (fix-up partials)
// belongs to this unit alone: gemm_bias_gelu_tf32_sk_workspace() bytes
int gemm_bias_gelu_tf32_sk(const float* A, const float* B, const float* bias, float* D, int M, int N, int K,
                           void* workspace, size_t workspace_bytes, cudaStream_t stream) {
#ifdef STC_HAVE_CUTLASS
  auto args = make_args_t<GemmSkFused>(A, B, bias, D, M, N, K);
  GemmSkFused gemm;
  if (GemmSkFused::get_workspace_size(args) > workspace_bytes || gemm.can_implement(args) != cutlass::Status::kSuccess)
    return 1;
  if (gemm.initialize(args, workspace, stream) != cutlass::Status::kSuccess) return 2;
  return gemm.run(stream) == cutlass::Status::kSuccess ? 0 : 2;
#else
  (void)A, (void)B, (void)bias, (void)D, (void)M, (void)N, (void)K, (void)workspace, (void)workspace_bytes, (void)stream;
  return 1;
#endif
}

long long gemm_bias_gelu_tf32_sk_workspace(int M, int N, int K) {
#ifdef STC_HAVE_CUTLASS
  auto args = make_args_t<GemmSkFused>(nullptr, nullptr, nullptr, nullptr, M, N, K);
  if (GemmSkFused::can_implement(args) != cutlass::Status::kSuccess) return -1;
  return static_cast<long long>(GemmSkFused::get_workspace_size(args));
#else
  (void)M, (void)N, (void)K;
  return -1;
#endif
}

// whether the fused path can run this shape (host-side check, no launch)
bool gemm_bias_gelu_supported(int M, int N, int K, size_t workspace_bytes) {
#ifdef STC_HAVE_CUTLASS
  auto args = make_args(nullptr, nullptr, nullptr, nullptr, M, N, K);
  return Gemm::get_workspace_size(args) <= workspace_bytes && Gemm::can_implement(args) == cutlass::Status::kSuccess;
#else
  (void)M, (void)N, (void)K, (void)workspace_bytes;
  return false;
#endif
}

}  // namespace stitch::gpu
