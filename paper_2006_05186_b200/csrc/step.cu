// bem_time_step: the whole time-domain operator step y = inverse(V(s_l) forward(x))
// (eq:omega_n P:436-441, eq:slphelm P:529-540 around the multi-frequency apply) as ONE
// library call, for host or device buffers.  The device part (K4 forward, K1/K2/K3
// apply, K4 inverse: ~25 launches) is captured once per (op, R) into a CUDA graph
// on an internal stream and replayed; host buffers are staged through the op's
// device time buffers with cudaMemcpyAsync (overlapping nothing else: the copies are
// the end-to-end cost a host caller pays).
#include <cstring>

#include "common.cuh"

namespace bem {

StepGraph::~StepGraph() {
  if (exec) cudaGraphExecDestroy(exec);
  if (own) cudaStreamDestroy(own);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e2) cudaEventDestroy(e2);
}

}  // namespace bem

using namespace bem;

extern "C" bem_status bem_time_step(bem_op oh, const bem_c128* x_time, bem_c128* y_time, double R,
                                    void* cuda_stream) {
  BEM_REQ(oh && x_time && y_time, "bem_time_step: NULL argument");
  BEM_REQ(R > 0.0 && R <= 1.0, "bem_time_step: R must lie in (0,1]");
  Op& op = oh->o;
  Tree& t = *op.tree;
  BEM_REQ(op.n_local == op.L, "bem_time_step: the operator must hold all L frequencies");
  for (int i = 0; i < op.n_local; ++i) BEM_REQ(op.local_l[i] == i, "bem_time_step: local_l must be 0..L-1 in order");
  DeviceGuard dg(t.device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int N = op.L - 1;
  const int64_t M = t.M;
  const size_t bytes = (size_t)op.L * M * 16;
  StepGraph& g = op.step;
  if (g.tx.n == 0) {
    BEM_CK(g.tx.alloc((size_t)op.L * M * 2)); BEM_CK(g.xf.alloc((size_t)op.L * M * 2));
    BEM_CK(g.yf.alloc((size_t)op.L * M * 2)); BEM_CK(g.ty.alloc((size_t)op.L * M * 2));
    BEM_CK(cudaStreamCreateWithFlags(&g.own, cudaStreamNonBlocking));
    BEM_CK(cudaEventCreateWithFlags(&g.e0, cudaEventDisableTiming));
    BEM_CK(cudaEventCreateWithFlags(&g.e1, cudaEventDisableTiming));
    BEM_CK(cudaEventCreateWithFlags(&g.e2, cudaEventDisableTiming));
  }
  // the op's time buffers are shared by every call: this call's H2D into g.tx must not
  // overtake the previous call's graph (or its D2H from g.ty), whatever stream it was on
  if (g.used) BEM_CK(cudaStreamWaitEvent(st, g.e2, 0));
  BEM_CK(cudaMemcpyAsync(g.tx.p, x_time, bytes, cudaMemcpyDefault, st));
  BEM_CK(cudaEventRecord(g.e0, st));
  BEM_CK(cudaStreamWaitEvent(g.own, g.e0, 0));
  auto body = [&](cudaStream_t s) -> bem_status {
    bem_status rs = fft_transform(g.tx.p, g.xf.p, M, N, R, false, s);
    if (rs == BEM_OK) rs = apply_launch(op, g.xf.p, g.yf.p, s);
    if (rs == BEM_OK) rs = fft_transform(g.yf.p, g.ty.p, M, N, R, true, s);
    return rs;
  };
  if (op.profile) {  // per-kernel event timers cannot live in a replayed graph: eager
    bem_status rs = body(g.own);
    if (rs != BEM_OK) return rs;
  } else {
    if (!g.exec || g.R != R) {
      if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
      // eager first pass: creates the transform plans and any lazily allocated
      // workspace outside the capture, and produces this call's result
      bem_status rs0 = body(g.own);
      if (rs0 != BEM_OK) return rs0;
      BEM_CK(cudaStreamSynchronize(g.own));
      cudaGraph_t graph = nullptr;
      BEM_CK(cudaStreamBeginCapture(g.own, cudaStreamCaptureModeThreadLocal));
      bem_status rs = body(g.own);
      cudaError_t ce = cudaStreamEndCapture(g.own, &graph);
      if (rs != BEM_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rs;
      }
      BEM_CK(ce);
      ce = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      BEM_CK(ce);
      g.R = R;
    } else {
      BEM_CK(cudaGraphLaunch(g.exec, g.own));
    }
  }
  BEM_CK(cudaEventRecord(g.e1, g.own));
  BEM_CK(cudaStreamWaitEvent(st, g.e1, 0));
  BEM_CK(cudaMemcpyAsync(y_time, g.ty.p, bytes, cudaMemcpyDefault, st));
  BEM_CK(cudaEventRecord(g.e2, st));
  g.used = true;
  return BEM_OK;
}
