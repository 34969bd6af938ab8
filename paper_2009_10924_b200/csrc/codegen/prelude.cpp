// Device-side helpers compiled into every NVRTC module, and small host
// formatting utilities for the generators.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>

#include "codegen/cg.hpp"

namespace stitch::gpu {

const std::string& device_prelude() {
  static const std::string src = R"CUDA(
// ---- stitch-b200 device prelude (sm_100a) ----
typedef long long i64;
typedef unsigned short f16_t;
#define FULL_MASK 0xffffffffu

__device__ __forceinline__ float h2f(f16_t h) { float f; asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h)); return f; }
__device__ __forceinline__ f16_t f2h(float f) { f16_t h; asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }

// tensor element <-> f32 value (stitch::DType: f32 / f16 / i32 / bool)
// Global loads are volatile asm so they keep their place relative to
// griddepcontrol.wait (also volatile): a kernel's graph-parameter loads are
// emitted before its PDL wait to overlap the previous kernel's drain, and a
// plain intrinsic / non-volatile asm load of read-only data may be sunk
// below the wait by the compiler (SASS showed ACQBULK first in every DIEN
// kernel).  STITCH_LD_FREE (an NVRTC define) restores free scheduling.
#ifdef STITCH_LD_FREE
#define STC_LD asm
#else
#define STC_LD asm volatile
#endif
__device__ __forceinline__ float ldv(const float* p, i64 i) {
  float v;
  STC_LD("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p + i));
  return v;
}
__device__ __forceinline__ float ldv(const f16_t* p, i64 i) {
  unsigned short h;
  STC_LD("ld.global.nc.u16 %0, [%1];" : "=h"(h) : "l"(p + i));
  return h2f(h);
}
__device__ __forceinline__ float ldv(const int* p, i64 i) {
  int v;
  STC_LD("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p + i));
  return (float)v;
}
__device__ __forceinline__ float ldv(const unsigned char* p, i64 i) {
  unsigned v;
  STC_LD("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p + i));
  return (v & 0xffu) ? 1.f : 0.f;
}
__device__ __forceinline__ void stv(float* p, i64 i, float v) { p[i] = v; }
__device__ __forceinline__ void stv(f16_t* p, i64 i, float v) { p[i] = f2h(v); }
__device__ __forceinline__ void stv(int* p, i64 i, float v) { p[i] = (int)roundf(v); }
__device__ __forceinline__ void stv(unsigned char* p, i64 i, float v) { p[i] = v != 0.f; }

// 128-bit streaming load of a graph parameter that does not allocate in L1
// (read-once data)
__device__ __forceinline__ float4 ld4(const float* p) {
  float4 r;
#ifdef STITCH_L2_256B
  STC_LD("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
#else
#ifdef STITCH_PARAM_NC
  STC_LD("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
#else
  // weak coherent load: ptxas keeps it ahead of griddepcontrol.wait where it
  // sinks .nc loads below it (bias+GELU 16.27 -> 15.70 us, others unchanged;
  // profiles/r01/param_load_path_ab.jsonl); STITCH_PARAM_NC restores .nc
  STC_LD("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
#endif
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
#endif
  return r;
}
// 128-bit load through L1 (data re-read by many threads, e.g. gamma/beta rows)
// Coherent loads (weak ld.global without .nc, no L1 allocation; =cg with
// STITCH_LDK_CG).  Two uses:
//  * tensors written by an EARLIER KERNEL of the graph (ld4k / ldvk /
//    ld4hk): under programmatic dependent launch this kernel starts before
//    its producer has finished, so such a tensor is not read-only for the
//    kernel's lifetime and must not be read through ld.global.nc -- ptxas
//    treats .nc loads as reads of immutable memory and may schedule them
//    above griddepcontrol.wait (observed: opaque placeholders);
//  * graph parameters that must be ISSUED before the PDL wait (ld4p /
//    ldvp, opaque_body): ptxas keeps coherent loads in front of a CTA
//    barrier, where it sinks .nc loads below the wait.
#ifdef STITCH_LDK_CG
#define STC_LDK "ld.global.cg"
#else
#define STC_LDK "ld.global.L1::no_allocate"
#endif
#define STC_LDK_V4(p, r) asm volatile(STC_LDK ".v4.f32 {%0,%1,%2,%3}, [%4];" \
                                      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p) : "memory")
__device__ __forceinline__ float4 ld4k(const float* p) { float4 r; STC_LDK_V4(p, r); return r; }
__device__ __forceinline__ float4 ld4p(const float* p) { float4 r; STC_LDK_V4(p, r); return r; }
__device__ __forceinline__ float ldvk(const float* p, i64 i) {
  float v;
  asm volatile(STC_LDK ".f32 %0, [%1];" : "=f"(v) : "l"(p + i) : "memory");
  return v;
}
__device__ __forceinline__ float ldvk(const f16_t* p, i64 i) {
  unsigned short h;
  asm volatile(STC_LDK ".u16 %0, [%1];" : "=h"(h) : "l"(p + i) : "memory");
  return h2f(h);
}
__device__ __forceinline__ float ldvk(const int* p, i64 i) {
  int v;
  asm volatile(STC_LDK ".s32 %0, [%1];" : "=r"(v) : "l"(p + i) : "memory");
  return (float)v;
}
__device__ __forceinline__ float ldvk(const unsigned char* p, i64 i) {
  unsigned v;
  asm volatile(STC_LDK ".u8 %0, [%1];" : "=r"(v) : "l"(p + i) : "memory");
  return (v & 0xffu) ? 1.f : 0.f;
}
template <typename T>
__device__ __forceinline__ float ldvp(const T* p, i64 i) { return ldvk(p, i); }
__device__ __forceinline__ float4 ld4c(const float* p) {
  float4 r;
  STC_LD("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
// 128-bit streaming (evict-first) store: outputs are written once and not
// re-read by this kernel (B200 A/B: profiles/r01/store_hint_sweep.jsonl)
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
#ifndef STITCH_ST_WB
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
#else
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
#endif
}

// 4 halves as one 64-bit access (f16 tensors, 4-aligned element index)
__device__ __forceinline__ float4 ld4h(const f16_t* p) {
  unsigned a, b;
  STC_LD("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
  return make_float4(h2f((f16_t)(a & 0xffffu)), h2f((f16_t)(a >> 16)), h2f((f16_t)(b & 0xffffu)), h2f((f16_t)(b >> 16)));
}
// coherent (L2, ld.global.cg) loads: the persistent template reads tensors
// written earlier in the same launch by other CTAs, which the non-coherent
// paths above may not
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); }
__device__ __forceinline__ void touch_l2(const void* p) {
  unsigned v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
}
// release-ordered add: the CTA's writes (ordered before it by a preceding
// __syncthreads) become visible at gpu scope no later than the count
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
#ifdef STITCH_PERSIST_SC_FENCE
  __threadfence();
  atomicAdd(p, v);
#else
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ldv_l2(const float* p, i64 i) { return __ldcg(p + i); }
__device__ __forceinline__ float ldv_l2(const f16_t* p, i64 i) { return h2f(__ldcg(p + i)); }
__device__ __forceinline__ float ldv_l2(const int* p, i64 i) { return (float)__ldcg(p + i); }
__device__ __forceinline__ float ldv_l2(const unsigned char* p, i64 i) { return __ldcg(p + i) ? 1.f : 0.f; }
__device__ __forceinline__ float4 ld4_l2(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4h_l2(const f16_t* p) {
  const uint2 q = __ldcg(reinterpret_cast<const uint2*>(p));
  return make_float4(h2f((f16_t)(q.x & 0xffffu)), h2f((f16_t)(q.x >> 16)), h2f((f16_t)(q.y & 0xffffu)), h2f((f16_t)(q.y >> 16)));
}
__device__ __forceinline__ float4 ld4hk(const f16_t* p) {
  unsigned a, b;
  asm volatile(STC_LDK ".v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p) : "memory");
  return make_float4(h2f((f16_t)(a & 0xffffu)), h2f((f16_t)(a >> 16)), h2f((f16_t)(b & 0xffffu)), h2f((f16_t)(b >> 16)));
}
__device__ __forceinline__ void st4h(f16_t* p, float x, float y, float z, float w) {
  const unsigned a = (unsigned)f2h(x) | ((unsigned)f2h(y) << 16), b = (unsigned)f2h(z) | ((unsigned)f2h(w) << 16);
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(a), "r"(b) : "memory");
}

// generic-address loads/stores (resident template): a unit's tensors may be
// graph buffers in global memory or slots in the CTA's shared memory, and
// every value read was written by this CTA before a CTA barrier
__device__ __forceinline__ float ldv_g(const float* p, i64 i) { return p[i]; }
__device__ __forceinline__ float ldv_g(const f16_t* p, i64 i) { return h2f(p[i]); }
__device__ __forceinline__ float ldv_g(const int* p, i64 i) { return (float)p[i]; }
__device__ __forceinline__ float ldv_g(const unsigned char* p, i64 i) { return p[i] ? 1.f : 0.f; }
__device__ __forceinline__ float4 ld4_g(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4h_g(const f16_t* p) {
  const uint2 q = *reinterpret_cast<const uint2*>(p);
  return make_float4(h2f((f16_t)(q.x & 0xffffu)), h2f((f16_t)(q.x >> 16)), h2f((f16_t)(q.y & 0xffffu)), h2f((f16_t)(q.y >> 16)));
}
__device__ __forceinline__ void st4_g(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4h_g(f16_t* p, float x, float y, float z, float w) {
  *reinterpret_cast<uint2*>(p) = make_uint2((unsigned)f2h(x) | ((unsigned)f2h(y) << 16), (unsigned)f2h(z) | ((unsigned)f2h(w) << 16));
}
template <typename T>
__device__ __forceinline__ T ldg_g(const T* p) { return *p; }

// e^x as 2^(x log2 e): one FMUL + MUFU.EX2.  Relative error <= |x| 2^-24
// (rounding of the product) + 2^-22 (ex2.approx) < 5.5e-6 for every finite
// result (|x| < 88.7) -- inside the 1e-5 elementwise band; results below
// FLT_MIN flush to 0 (absolute error < 1.2e-38).  STITCH_FAST_EXP=0 emits expf.
__device__ __forceinline__ float exp_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.44269504088896341f));
  return y;
}

// per-op rounding to the node dtype (src/sim.cpp:67-75 semantics)
__device__ __forceinline__ float rnd_f16(float x) { return h2f(f2h(x)); }
__device__ __forceinline__ float rnd_i32(float x) { return (float)(int)roundf(x); }
__device__ __forceinline__ float rnd_bool(float x) { return x != 0.f ? 1.f : 0.f; }

// std::max / std::min argument order (NaN behaviour of the reference)
__device__ __forceinline__ float op_max(float a, float b) { return a < b ? b : a; }
__device__ __forceinline__ float op_min(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ float op_rsqrt(float a) { return 1.0f / sqrtf(a); }
// a / b given r = RN(1/b), r normal: Markstein's FMA correction yields the
// correctly rounded quotient (same bits as IEEE division)
__device__ __forceinline__ float div_rcp(float a, float b, float r) {
  const float q = a * r;
  const float e = __fmaf_rn(-q, b, a);
  return __fmaf_rn(e, r, q);
}
// compensated (Kahan) f32 accumulation; the pair is folded to f64 before the
// cross-thread tree, so partial sums keep ~f64 accuracy at f32 issue cost
__device__ __forceinline__ void kahan_add(float& s, float& c, float x) {
  const float y = x - c;
  const float t = s + y;
  c = (t - s) - y;
  s = t;
}

// butterfly over `width` lanes (power of two <= 32): every lane gets the result
__device__ __forceinline__ double bfly_sum(double v, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ float bfly_max(float v, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) v = op_max(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}

// in-graph kernel timeline (STITCH_TRACE=1 builds): per kernel slot k,
// [2k] = earliest CTA entry, [2k+1] = latest CTA exit (%globaltimer, ns)
#ifdef STITCH_TRACE
__device__ unsigned long long stc_trace_[2 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef STITCH_TRACE_CTAS  // per-CTA slots: k * CTAS + CTA (CTAs past CTAS fold into CTA 0's)
#define STC_SLOT(k) ((k) * STITCH_TRACE_CTAS + (blockIdx.x < STITCH_TRACE_CTAS ? blockIdx.x : 0))
#else
#define STC_SLOT(k) (k)
#endif
#define STC_TRACE_BEGIN(k) do { if (threadIdx.x == 0) atomicMin(&stc_trace_[2 * STC_SLOT(k)], gtimer()); } while (0)
#define STC_TRACE_END(k) do { __syncthreads(); if (threadIdx.x == 0) atomicMax(&stc_trace_[2 * STC_SLOT(k) + 1], gtimer()); } while (0)
#define STC_TRACE_STAMP_END(k) do { if (threadIdx.x == 0) atomicMax(&stc_trace_[2 * STC_SLOT(k) + 1], gtimer()); } while (0)
#else
#define STC_TRACE_BEGIN(k) do {} while (0)
#define STC_TRACE_END(k) do {} while (0)
#define STC_TRACE_STAMP_END(k) do {} while (0)
#endif

// programmatic dependent launch (PDL): no-ops unless launched with the
// programmatic-stream-serialization attribute
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- TMA bulk copies + mbarriers (sm_90+; the regional pipeline) ----
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile("{\n .reg .pred P1;\n LAB_WAIT:\n"
               " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}" :: "r"(smem_addr(b)), "r"(parity) : "memory");
}
// global -> shared bulk copy (TMA engine, no tensor map), completes on `b`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)) : "memory");
}
// order this CTA's generic-proxy smem accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// ---- thread-block clusters (regional-cluster template: one long row per cluster)
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// f64 in the shared memory of cluster CTA `rank` (DSMEM)
__device__ __forceinline__ double ld_dsmem_f64(const double* p, unsigned rank) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

// remote push (resident template): the f64 `v` into cluster CTA `rank`'s
// shared memory at (our address of) `dst`, completing `bytes` on that CTA's
// mbarrier `b` -- a one-way signal instead of a cluster-wide barrier
__device__ __forceinline__ void st_async_f64(double* dst, double v, unsigned long long* b, unsigned rank) {
  unsigned rd, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_addr(dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_addr(b)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(rd), "d"(v), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* b, unsigned parity) {
  asm volatile("{\n .reg .pred P1;\n LAB_WAITC:\n"
               " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
               " @P1 bra DONEC;\n bra LAB_WAITC;\n DONEC:\n}" :: "r"(smem_addr(b)), "r"(parity) : "memory");
}

// run_program fault report: first fault wins (code 1 race, 2 global OOB, 3 shared OOB)
__device__ __forceinline__ void sim_fault(unsigned* f, unsigned code, i64 where) {
  if (atomicCAS(f, 0u, code) == 0u) {
    f[1] = (unsigned)(where & 0xffffffff);
    f[2] = threadIdx.x;
    f[3] = blockIdx.x;
  }
}

// Grid-wide barrier for cooperative (co-resident) launches.  bar[0] counts
// arrivals, bar[1] is the generation; both start at zero and bar[0] returns
// to zero after every barrier, so the scratch word can be reused forever.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}
)CUDA";
  return src;
}

std::string c_float(double v) {
  const float f = static_cast<float>(v);
  if (std::isnan(f)) return "__int_as_float(0x7fc00000)";
  if (std::isinf(f)) return f > 0 ? "__int_as_float(0x7f800000)" : "__int_as_float(0xff800000)";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.9ef", static_cast<double>(f));  // round-trips exactly
  return buf;
}

const char* c_type(DType d) {
  switch (d) {
    case DType::F32: return "float";
    case DType::F16: return "f16_t";
    case DType::I32: return "int";
    case DType::Bool: return "unsigned char";
  }
  return "float";
}

int64_t algorithmic_bytes(const CompGraph& g, const std::vector<int>& vertices) {
  std::set<int> in(vertices.begin(), vertices.end());
  std::set<int> ext_in, ext_out;
  for (int v : vertices) {
    for (int o : g.node(v).operands)
      if (!in.count(o) && g.node(o).kind != OpKind::Constant) ext_in.insert(o);
    if (g.is_output(v)) ext_out.insert(v);
  }
  for (const auto& n : g.nodes)
    if (!in.count(n.id))
      for (int o : n.operands)
        if (in.count(o)) ext_out.insert(o);
  int64_t b = 0;
  for (int t : ext_in) b += g.node(t).shape.byte_size();
  for (int t : ext_out) b += g.node(t).shape.byte_size();
  return b;
}

}  // namespace stitch::gpu
