// Probe (diagnostics): when does a CUDA-graph kernel node with several
// predecessors launch under programmatic dependent launch?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/pdl_edge_probe.cu -o /tmp/pdl_edge_probe -lcuda
//
// A spins ~8 us and triggers dependents at entry; B is a short kernel on a
// second lane that finished long before; C depends on A (same lane) and,
// in some variants, on B (cross lane).  C records its first-CTA entry time;
// "lead" = A's end - C's entry (positive: C launched while A still ran).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin(unsigned long long* ts, int slot, int ns, int trigger_early) {
  if (trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) ts[2 * slot] = t0;
  while (gt() - t0 < static_cast<unsigned long long>(ns)) {
  }
  __syncthreads();
  if (threadIdx.x == 0) ts[2 * slot + 1] = gt();
}

__global__ void probe(unsigned long long* ts, int slot) {
  unsigned long long t0 = gt();  // entry, before the wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    ts[2 * slot] = t0;
    ts[2 * slot + 1] = gt();
  }
}

static void launch(void (*k)(unsigned long long*, int), cudaStream_t s, bool pdl, unsigned long long* ts, int slot) {
  cudaLaunchConfig_t c{};
  c.gridDim = dim3(1);
  c.blockDim = dim3(128);
  c.stream = s;
  cudaLaunchAttribute a{};
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  c.attrs = &a;
  c.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&c, k, ts, slot));
}

static void launch_spin(cudaStream_t s, bool pdl, unsigned long long* ts, int slot, int ns, int early) {
  cudaLaunchConfig_t c{};
  c.gridDim = dim3(1);
  c.blockDim = dim3(128);
  c.stream = s;
  cudaLaunchAttribute a{};
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  c.attrs = &a;
  c.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&c, spin, ts, slot, ns, early));
}

int main() {
  unsigned long long* ts = nullptr;
  CK(cudaMalloc(&ts, 64 * sizeof(unsigned long long)));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t ev, fork;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  const char* names[] = {"same-lane only (A->C)", "A->C + cross-lane B->C (B done early)",
                         "A->C + cross-lane B->C, B without PDL", "A->C + B->C, B on same lane before A",
                         "chain A->A2->C (C waits on grand-parent)",
                         "A only on the other lane (cross-lane A->C, P->C same lane)",
                         "fork P->{A, A2 on lane 2} -> C (join)",
                         "one lane A(8us)->A2->B->C: C three levels behind the running A",
                         "one lane A(8us)->A2->C: C two levels behind the running A"};
  for (int variant = 0; variant < 9; ++variant) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s1, cudaStreamCaptureModeThreadLocal));
    // slot 0: P (a predecessor so A itself launches from a PDL edge), 1: A, 2: B, 3: C, 4: A2
    launch_spin(s1, false, ts, 0, 1000, 1);
    if (variant == 1 || variant == 2) {
      CK(cudaEventRecord(fork, s1));
      CK(cudaStreamWaitEvent(s2, fork, 0));
      launch_spin(s2, variant == 1, ts, 2, 200, 1);
      CK(cudaEventRecord(ev, s2));
    }
    if (variant == 3) launch_spin(s1, true, ts, 2, 200, 1);
    if (variant == 5 || variant == 6) {
      CK(cudaEventRecord(fork, s1));
      CK(cudaStreamWaitEvent(s2, fork, 0));
      launch_spin(s2, true, ts, 1, 8000, 1);
      CK(cudaEventRecord(ev, s2));
      if (variant == 6) launch_spin(s1, true, ts, 4, 3000, 1);
      CK(cudaStreamWaitEvent(s1, ev, 0));
    } else {
      launch_spin(s1, true, ts, 1, 8000, 1);
    }
    if (variant == 4) launch_spin(s1, true, ts, 4, 3000, 1);
    if (variant == 7 || variant == 8) launch_spin(s1, true, ts, 4, 300, 1);
    if (variant == 7) launch_spin(s1, true, ts, 2, 300, 1);
    if (variant == 1 || variant == 2) CK(cudaStreamWaitEvent(s1, ev, 0));
    launch(probe, s1, true, ts, 3);
    CK(cudaStreamEndCapture(s1, &g));
    size_t ne = 0;
    CK(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));
    std::vector<cudaGraphNode_t> from(ne), to(ne);
    std::vector<cudaGraphEdgeData> ed(ne);
    CK(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne));
    int prog = 0;
    for (auto& e : ed) prog += e.type == cudaGraphDependencyTypeProgrammatic;
    cudaGraphExec_t x;
    CK(cudaGraphInstantiate(&x, g, 0));
    double lead = 0, wait_gap = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 3; ++r) {
      CK(cudaMemsetAsync(ts, 0, 64 * sizeof(unsigned long long), s1));
      CK(cudaGraphLaunch(x, s1));
      CK(cudaStreamSynchronize(s1));
      unsigned long long h[16];
      CK(cudaMemcpy(h, ts, sizeof h, cudaMemcpyDeviceToHost));
      // lead is measured against the running head A (slot 1) for 7/8
      const unsigned long long last_end = variant == 4 ? h[9] : h[3];
      if (r >= 3) {
        lead += (static_cast<double>(last_end) - static_cast<double>(h[6])) / 1e3;
        wait_gap += (static_cast<double>(h[7]) - static_cast<double>(last_end)) / 1e3;
      }
    }
    std::printf("{\"variant\": \"%s\", \"edges\": %zu, \"programmatic_edges\": %d, \"C_entry_lead_us\": %.2f, "
                "\"C_wait_return_after_pred_end_us\": %.2f}\n",
                names[variant], ne, prog, lead / reps, wait_gap / reps);
    CK(cudaGraphExecDestroy(x));
    CK(cudaGraphDestroy(g));
  }
  return 0;
}
