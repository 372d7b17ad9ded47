// Multi-GPU frequency sharding over NCCL (Remark P:1607-1614:
// the systems of different frequencies decouple).
//
// Layout of a G-rank run (rank g):
//   * frequency classes {0} and {j, L-j} (j = 1..) stay whole on one rank -- K1
//     shares one exp/sincos per conjugate pair --, class i on rank i mod G
//     (shard_frequencies below == paper_2006_05186_b200/dist.py, tested);
//     the op of rank g holds exactly that local frequency list, in that order;
//   * time-domain data are DOF-sharded: rank g owns panels [M g/G, M (g+1)/G).
// The time <-> frequency transpose is ONE all-to-all per direction, grouped
// ncclSend / ncclRecv of packed chunks:
//   forward: K4 writes frequency row l of this rank's DOF columns straight into
//            its slot of the packed send buffer (row table in the kernel
//            parameters: transform + pack in one pass), NCCL exchanges the
//            [L_h][M_g] chunks, a strided 2-D copy per source rank places the
//            received [L_g][M_h] chunks into the [L_g][M] frequency shard;
//   inverse: the mirror image (2-D copies pack [L_g][M_h] chunks, NCCL, K4
//            reads each frequency row from its slot of the receive buffer).
// The frequency-domain apply itself needs no collective.  NCCL is loaded at
// run time (dlopen "libnccl.so.2": the copy torch already loaded, else the
// system one), so the library still loads where NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace bem {
namespace {

struct Nccl {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
    n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
    n.send = (decltype(n.send))dlsym(h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
    n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
    n.errorString = (decltype(n.errorString))dlsym(h, "ncclGetErrorString");
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.groupStart && n.groupEnd && n.send && n.recv &&
           n.allReduce && n.errorString;
  });
  return n;
}

#define BEM_NC(call)                                                                     \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      bem::set_error("NCCL error at %s:%d: %s", __FILE__, __LINE__, nccl().errorString(r_)); \
      return BEM_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

}  // namespace

// Frequency shard of every rank: owner[l] = rank holding l, slot[l] = its row in that
// rank's local list.  Classes {0}, {j, L-j} dealt round-robin (class i on rank i mod G, a
// rank's classes in increasing i), at least one class per rank.
bool shard_frequencies(int L, int G, std::vector<int>& owner, std::vector<int>& slot,
                       std::vector<std::vector<int>>* lists) {
  std::vector<std::vector<int>> cls;
  cls.push_back({0});
  for (int j = 1; j <= L / 2; ++j) {
    if (L - j != j) cls.push_back({j, L - j});
    else cls.push_back({j});
  }
  const int nc = (int)cls.size();
  if (G < 1 || G > nc) return false;
  owner.assign(L, -1);
  slot.assign(L, -1);
  if (lists) lists->assign(G, {});
  // class i -> rank i mod G: every rank holds an even sample of the frequency circle, so the
  // underflow cutoffs (K1 / K3 leave out most work of the strongly damped frequencies) take
  // the same share from every rank
  for (int g = 0; g < G; ++g) {
    int k = 0;
    for (int i = g; i < nc; i += G)
      for (int l : cls[i]) {
        owner[l] = g;
        slot[l] = k++;
        if (lists) (*lists)[g].push_back(l);
      }
  }
  return true;
}

}  // namespace bem

struct bem_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  bem::DBuf<double> red;  // small device buffer for the solve statistics
};

namespace bem {

// Per-op state of the sharded transposes (allocated at the first call, reused).
struct ShardWs {
  int G = 0, rank = -1, L = 0;
  int64_t M = 0, b = 0, Mg = 0;
  std::vector<int> owner, slot, Lh, cumL;     // per frequency / per rank
  std::vector<int64_t> bh, Mh, cumM;          // DOF ranges per rank, prefix sums of M_h
  DBuf<double> send, recv, xf, yf;            // [L][M_g] packed, [L][M_g] packed, [L_g][M] x2
  std::vector<const double2*> fwd_rows, inv_rows;
};

namespace {

std::mutex g_ws_mu;
std::vector<std::pair<const Op*, ShardWs*>> g_ws;

bem_status shard_ws(Op& op, bem_comm c, ShardWs** out) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (auto& e : g_ws)
    if (e.first == &op && e.second->G == c->nranks && e.second->rank == c->rank) { *out = e.second; return BEM_OK; }
  const int L = op.L, G = c->nranks, g = c->rank;
  const int64_t M = op.tree->M;
  auto* w = new ShardWs();
  std::vector<std::vector<int>> lists;
  if (!shard_frequencies(L, G, w->owner, w->slot, &lists)) {
    delete w;
    set_error("sharded step: %d ranks but only %d frequency classes", G, L / 2 + 1);
    return BEM_EINVAL;
  }
  if ((int)op.local_l.size() != (int)lists[g].size() || !std::equal(lists[g].begin(), lists[g].end(), op.local_l.begin())) {
    delete w;
    set_error("sharded step: the op's local frequencies are not rank %d's shard of %d (dist.shard_frequencies)", g, G);
    return BEM_EINVAL;
  }
  w->G = G; w->rank = g; w->L = L; w->M = M;
  w->Lh.resize(G); w->cumL.assign(G + 1, 0); w->bh.resize(G); w->Mh.resize(G); w->cumM.assign(G + 1, 0);
  for (int h = 0; h < G; ++h) {
    w->Lh[h] = (int)lists[h].size();
    w->cumL[h + 1] = w->cumL[h] + w->Lh[h];
    w->bh[h] = M * h / G;
    w->Mh[h] = M * (h + 1) / G - w->bh[h];
    w->cumM[h + 1] = w->cumM[h] + w->Mh[h];
  }
  w->b = w->bh[g]; w->Mg = w->Mh[g];
  // packed buffers serve both directions: [L][M_g] rows by owner, and [L_g][M] chunks by DOF range
  const size_t fs = (size_t)w->Lh[g] * M * 2, pk = std::max((size_t)L * w->Mg * 2, fs);
  if (w->send.alloc(std::max<size_t>(pk, 2)) != cudaSuccess || w->recv.alloc(std::max<size_t>(pk, 2)) != cudaSuccess ||
      w->xf.alloc(std::max<size_t>(fs, 2)) != cudaSuccess || w->yf.alloc(std::max<size_t>(fs, 2)) != cudaSuccess) {
    delete w;
    set_error("sharded step: workspace allocation failed");
    return BEM_ENOMEM;
  }
  w->fwd_rows.resize(L);
  w->inv_rows.resize(L);
  for (int l = 0; l < L; ++l) {
    const int64_t row = (int64_t)w->cumL[w->owner[l]] + w->slot[l];  // packed row of frequency l
    w->fwd_rows[l] = (const double2*)w->send.p + row * w->Mg;
    w->inv_rows[l] = (const double2*)w->recv.p + row * w->Mg;
  }
  g_ws.push_back({&op, w});
  *out = w;
  return BEM_OK;
}

}  // namespace

void shard_ws_release(const Op* op) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (size_t i = 0; i < g_ws.size();) {
    if (g_ws[i].first == op) { delete g_ws[i].second; g_ws.erase(g_ws.begin() + i); }
    else ++i;
  }
}

// The two transposes, split into the per-rank packing steps and the exchange, so that the
// NCCL path and the single-process check (bem_debug_sharded_step) share the packing code.
// forward, rank g: K4 over this rank's DOF columns, frequency row l stored into its slot
// (owner(l), slot(l)) of the packed send buffer
static bem_status fwd_pack(ShardWs* w, const double* x_time, double R, cudaStream_t st) {
  return fft_transform_rows(x_time, nullptr, w->Mg, w->L - 1, R, false, st, w->fwd_rows.data(), 2);
}
// forward exchange: rank g's chunk for h = rows cumL[h].. of its send buffer ([L_h][M_g]);
// rank h stores it at cumM[g] * L_h in its receive buffer
static double* fwd_send_chunk(ShardWs* w, int h) { return w->send.p + (size_t)w->cumL[h] * w->Mg * 2; }
static size_t fwd_chunk_n(ShardWs* from, ShardWs* to) { return (size_t)to->Lh[to->rank] * from->Mg * 2; }
static double* fwd_recv_chunk(ShardWs* w, int g) { return w->recv.p + (size_t)w->cumM[g] * w->Lh[w->rank] * 2; }
// forward unpack: [L_g][M_h] chunks -> columns [b_h, b_h + M_h) of the [L_g][M] frequency shard
static bem_status fwd_unpack(ShardWs* w, cudaStream_t st) {
  const int g = w->rank;
  for (int h = 0; h < w->G; ++h)
    if (w->Mh[h] > 0 && w->Lh[g] > 0)
      BEM_CK(cudaMemcpy2DAsync(w->xf.p + (size_t)w->bh[h] * 2, (size_t)w->M * 16,
                               w->recv.p + (size_t)w->cumM[h] * w->Lh[g] * 2, (size_t)w->Mh[h] * 16,
                               (size_t)w->Mh[h] * 16, (size_t)w->Lh[g], cudaMemcpyDeviceToDevice, st));
  return BEM_OK;
}
// inverse pack: columns [b_h, b_h + M_h) of yf -> packed [L_g][M_h] chunk for rank h
static bem_status inv_pack(ShardWs* w, const double2* yf, cudaStream_t st) {
  const int g = w->rank;
  for (int h = 0; h < w->G; ++h)
    if (w->Mh[h] > 0 && w->Lh[g] > 0)
      BEM_CK(cudaMemcpy2DAsync(w->send.p + (size_t)w->cumM[h] * w->Lh[g] * 2, (size_t)w->Mh[h] * 16,
                               (const double*)yf + (size_t)w->bh[h] * 2, (size_t)w->M * 16, (size_t)w->Mh[h] * 16,
                               (size_t)w->Lh[g], cudaMemcpyDeviceToDevice, st));
  return BEM_OK;
}
static double* inv_send_chunk(ShardWs* w, int h) { return w->send.p + (size_t)w->cumM[h] * w->Lh[w->rank] * 2; }
static size_t inv_chunk_n(ShardWs* from, ShardWs* to) { return (size_t)from->Lh[from->rank] * to->Mg * 2; }
static double* inv_recv_chunk(ShardWs* w, int g) { return w->recv.p + (size_t)w->cumL[g] * w->Mg * 2; }
// inverse unpack: K4 reading frequency row l from its slot of the receive buffer
static bem_status inv_unpack(ShardWs* w, double* y_time, double R, cudaStream_t st) {
  return fft_transform_rows(nullptr, y_time, w->Mg, w->L - 1, R, true, st, w->inv_rows.data(), 1);
}

// x_time [L][M_g] (this rank's DOFs, device) -> xf [L_g][M] (this rank's frequencies)
bem_status shard_forward(Op& op, bem_comm c, const double* x_time, double R, double2** xf, cudaStream_t st) {
  ShardWs* w = nullptr;
  bem_status rs = shard_ws(op, c, &w);
  if (rs != BEM_OK) return rs;
  const int G = w->G;
  rs = fwd_pack(w, x_time, R, st);
  if (rs != BEM_OK) return rs;
  Nccl& n = nccl();
  BEM_NC(n.groupStart());
  for (int h = 0; h < G; ++h) {
    BEM_NC(n.send(fwd_send_chunk(w, h), (size_t)w->Lh[h] * w->Mg * 2, ncclDouble, h, c->comm, st));
    BEM_NC(n.recv(fwd_recv_chunk(w, h), (size_t)w->Lh[w->rank] * w->Mh[h] * 2, ncclDouble, h, c->comm, st));
  }
  BEM_NC(n.groupEnd());
  rs = fwd_unpack(w, st);
  *xf = (double2*)w->xf.p;
  return rs;
}

// yf [L_g][M] (this rank's frequencies) -> y_time [L][M_g] (this rank's DOFs)
bem_status shard_inverse(Op& op, bem_comm c, const double2* yf, double R, double* y_time, cudaStream_t st) {
  ShardWs* w = nullptr;
  bem_status rs = shard_ws(op, c, &w);
  if (rs != BEM_OK) return rs;
  const int G = w->G;
  rs = inv_pack(w, yf, st);
  if (rs != BEM_OK) return rs;
  Nccl& n = nccl();
  BEM_NC(n.groupStart());
  for (int h = 0; h < G; ++h) {
    BEM_NC(n.send(inv_send_chunk(w, h), (size_t)w->Lh[w->rank] * w->Mh[h] * 2, ncclDouble, h, c->comm, st));
    BEM_NC(n.recv(inv_recv_chunk(w, h), (size_t)w->Lh[h] * w->Mg * 2, ncclDouble, h, c->comm, st));
  }
  BEM_NC(n.groupEnd());
  return inv_unpack(w, y_time, R, st);
}

// G ranks in one process on one device, the exchange done by device copies instead of
// NCCL (same packing code): the multi-rank transposes checked where only one GPU exists.
bem_status sharded_step_virtual(int G, Op** ops, const double* const* x, double* const* y, double R,
                                cudaStream_t st) {
  std::vector<bem_comm_s> cs(G);
  std::vector<ShardWs*> w(G, nullptr);
  for (int g = 0; g < G; ++g) {
    cs[g].nranks = G; cs[g].rank = g; cs[g].device = ops[g]->tree->device;
    bem_status rs = shard_ws(*ops[g], &cs[g], &w[g]);
    if (rs != BEM_OK) return rs;
  }
  for (int g = 0; g < G; ++g) {
    bem_status rs = fwd_pack(w[g], x[g], R, st);
    if (rs != BEM_OK) return rs;
  }
  for (int g = 0; g < G; ++g)
    for (int h = 0; h < G; ++h)
      BEM_CK(cudaMemcpyAsync(fwd_recv_chunk(w[h], g), fwd_send_chunk(w[g], h), fwd_chunk_n(w[g], w[h]) * 8,
                             cudaMemcpyDeviceToDevice, st));
  for (int g = 0; g < G; ++g) {
    bem_status rs = fwd_unpack(w[g], st);
    if (rs == BEM_OK) rs = apply_launch(*ops[g], w[g]->xf.p, w[g]->yf.p, st);
    if (rs == BEM_OK) rs = inv_pack(w[g], (const double2*)w[g]->yf.p, st);
    if (rs != BEM_OK) return rs;
  }
  for (int g = 0; g < G; ++g)
    for (int h = 0; h < G; ++h)
      BEM_CK(cudaMemcpyAsync(inv_recv_chunk(w[h], g), inv_send_chunk(w[g], h), inv_chunk_n(w[g], w[h]) * 8,
                             cudaMemcpyDeviceToDevice, st));
  for (int g = 0; g < G; ++g) {
    bem_status rs = inv_unpack(w[g], y[g], R, st);
    if (rs != BEM_OK) return rs;
  }
  return BEM_OK;
}

bem_status shard_yf(Op& op, bem_comm c, double2** yf) {
  ShardWs* w = nullptr;
  bem_status rs = shard_ws(op, c, &w);
  if (rs != BEM_OK) return rs;
  *yf = (double2*)w->yf.p;
  return BEM_OK;
}

// element-wise max (first nmax doubles) and sum (next nsum) over the ranks, in place on the device
bem_status comm_allreduce(bem_comm c, double* dev, int nmax, int nsum, cudaStream_t st) {
  Nccl& n = nccl();
  if (nmax > 0) BEM_NC(n.allReduce(dev, dev, (size_t)nmax, ncclDouble, ncclMax, c->comm, st));
  if (nsum > 0) BEM_NC(n.allReduce(dev + nmax, dev + nmax, (size_t)nsum, ncclDouble, ncclSum, c->comm, st));
  return BEM_OK;
}

double* comm_scratch(bem_comm c) { return c->red.p; }

bem_status comm_check(bem_comm c, const Op& op, int64_t M_loc) {
  BEM_REQ(c->comm != nullptr, "bem_comm: not initialised");
  BEM_REQ(c->device == op.tree->device, "bem_comm: communicator on device %d, op on device %d", c->device,
          op.tree->device);
  const int64_t M = op.tree->M;
  const int64_t Mg = M * (c->rank + 1) / c->nranks - M * c->rank / c->nranks;
  BEM_REQ(M_loc == Mg, "sharded call: M_loc = %lld, rank %d of %d owns %lld panels", (long long)M_loc, c->rank,
          c->nranks, (long long)Mg);
  return BEM_OK;
}

}  // namespace bem

using namespace bem;

extern "C" bem_status bem_comm_unique_id(void* id_out) {
  BEM_REQ(id_out, "bem_comm_unique_id: NULL argument");
  if (!nccl().ok) {
    set_error("bem_comm_unique_id: libnccl.so.2 could not be loaded");
    return BEM_ENCCL;
  }
  ncclUniqueId id;
  BEM_NC(nccl().getUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return BEM_OK;
}

extern "C" bem_status bem_comm_init(const void* id, int32_t nranks, int32_t rank, int32_t device, bem_comm* out) {
  BEM_REQ(id && out, "bem_comm_init: NULL argument");
  BEM_REQ(nranks >= 1 && rank >= 0 && rank < nranks, "bem_comm_init: rank %d of %d", rank, nranks);
  *out = nullptr;
  if (!nccl().ok) {
    set_error("bem_comm_init: libnccl.so.2 could not be loaded");
    return BEM_ENCCL;
  }
  DeviceGuard dg(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* c = new bem_comm_s();
  c->nranks = nranks; c->rank = rank; c->device = device;
  const ncclResult_t r = nccl().commInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    set_error("bem_comm_init: ncclCommInitRank: %s", nccl().errorString(r));
    delete c;
    return BEM_ENCCL;
  }
  if (c->red.alloc(8) != cudaSuccess) {
    nccl().commDestroy(c->comm);
    delete c;
    set_error("bem_comm_init: allocation failed");
    return BEM_ENOMEM;
  }
  *out = c;
  return BEM_OK;
}

extern "C" bem_status bem_comm_destroy(bem_comm c) {
  if (!c) return BEM_OK;
  DeviceGuard dg(c->device);
  if (c->comm) nccl().commDestroy(c->comm);
  delete c;
  return BEM_OK;
}

extern "C" bem_status bem_shard_frequencies(int32_t L, int32_t G, int32_t* owner, int32_t* slot) {
  BEM_REQ(L >= 1 && owner && slot, "bem_shard_frequencies: bad arguments");
  std::vector<int> o, s;
  BEM_REQ(shard_frequencies(L, G, o, s, nullptr), "bem_shard_frequencies: G = %d ranks for %d classes", G, L / 2 + 1);
  for (int l = 0; l < L; ++l) { owner[l] = o[l]; slot[l] = s[l]; }
  return BEM_OK;
}

extern "C" bem_status bem_time_step_sharded(bem_op oh, const bem_c128* x_loc, bem_c128* y_loc, int64_t M_loc,
                                            double R, bem_comm c, void* cuda_stream) {
  BEM_REQ(oh && x_loc && y_loc && c, "bem_time_step_sharded: NULL argument");
  BEM_REQ(R > 0.0 && R <= 1.0, "bem_time_step_sharded: R must lie in (0,1]");
  Op& op = oh->o;
  bem_status rs = comm_check(c, op, M_loc);
  if (rs != BEM_OK) return rs;
  DeviceGuard dg(op.tree->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  double2 *xf = nullptr, *yf = nullptr;
  rs = shard_forward(op, c, (const double*)x_loc, R, &xf, st);
  if (rs == BEM_OK) rs = shard_yf(op, c, &yf);
  if (rs == BEM_OK) rs = apply_launch(op, (const double*)xf, (double*)yf, st);
  if (rs == BEM_OK) rs = shard_inverse(op, c, yf, R, (double*)y_loc, st);
  return rs;
}

extern "C" bem_status bem_debug_sharded_step(int32_t G, bem_op* ops, const bem_c128* const* x_loc,
                                             bem_c128* const* y_loc, double R, void* cuda_stream) {
  BEM_REQ(G >= 1 && ops && x_loc && y_loc, "bem_debug_sharded_step: bad arguments");
  std::vector<Op*> o(G);
  std::vector<const double*> x(G);
  std::vector<double*> y(G);
  for (int g = 0; g < G; ++g) {
    BEM_REQ(ops[g] && x_loc[g] && y_loc[g], "bem_debug_sharded_step: NULL entry %d", g);
    o[g] = &ops[g]->o;
    BEM_REQ(o[g]->tree->device == o[0]->tree->device, "bem_debug_sharded_step: ops on different devices");
    x[g] = (const double*)x_loc[g];
    y[g] = (double*)y_loc[g];
  }
  DeviceGuard dg(o[0]->tree->device);
  return sharded_step_virtual(G, o.data(), x.data(), y.data(), R, (cudaStream_t)cuda_stream);
}
