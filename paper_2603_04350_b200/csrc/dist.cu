// dist.cu -- multi-GPU plumbing of the sweep:
// the mode-slab / time-slab partition, the all-to-all message schedules between the two
// layouts, and their execution with NCCL point-to-point calls (NCCL is loaded at run time,
// so the single-GPU library has no NCCL dependency).
//
// Partition (P ranks, nt % P == 0):
//   * time slab of rank r: slices [r nt/P, (r+1) nt/P) of a space-time vector, full
//     spatial slices -- where the space-local stage 3 (N-hat = V N(V u-hat)) runs;
//   * mode slab of rank r: a contiguous range [off_r, off_r + len_r) of the padded spectral
//     entries of every slice (whole padded x-lines for dim >= 2, mode pairs for dim 1), all
//     nt slices -- where the time-local K1 (residual, alpha-circulant preconditioner,
//     update) runs.  In the DST basis every spatial mode is an independent length-nt
//     problem ("naturally parallelizable"), so K1 needs no
//     communication; norms and GMRES inner products are partial sums + one allreduce.
// A schedule is plain data (a list of messages), so the same list is executed by NCCL
// here and by torch.distributed (gloo) in the CPU tests (tests/test_dist_cpu.py).  A host
// communicator (expd_host_comm_create) runs the device plan's exchanges through host
// staging buffers and a caller transport instead of NCCL: the multi-rank plan can then be
// exercised by several processes sharing one GPU (tests/test_gpu_multirank.py), whose
// kernels never wait on one another -- the hosts exchange the data.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "../../include/expd.h"
#include "expd_internal.h"

namespace expd {

bool dist_layout(const Geom& g, int nt, int rank, int nranks, DistLayout* L) {
  if (nranks < 1 || nranks > EXPD_MAX_RANKS || rank < 0 || rank >= nranks || nt % nranks != 0) return false;
  L->rank = rank;
  L->nranks = nranks;
  L->nt = nt;
  L->npad = g.npad;
  L->unit = g.dim >= 2 ? g.M : 2;  // whole padded x-lines (dim >= 2) or mode pairs (dim 1)
  const long units = g.npad / L->unit;
  if (units < nranks) return false;
  const long base = units / nranks, rem = units % nranks;
  long off = 0;
  for (int q = 0; q < nranks; ++q) {
    const long u = base + (q < rem ? 1 : 0);
    L->mode_off[q] = off * L->unit;
    L->mode_len[q] = u * L->unit;
    off += u;
    L->t0[q] = q * (nt / nranks);
    L->ntl[q] = nt / nranks;
  }
  return true;
}

// Messages of one all-to-all between the layouts, in the order both sides post them.
//   MODE_TO_TIME: src = mode slab [nt][len_r], dst = time slab [ntl_r][npad];
//   TIME_TO_MODE: src = time slab [ntl_r][npad], dst = mode slab [nt + shift][len_r],
//                 global slice t lands in dst slice t + shift.
// Self messages (peer == rank) are local copies.
void a2a_schedule(const DistLayout& L, int dir, int shift, std::vector<A2AMsg>& sends, std::vector<A2AMsg>& recvs) {
  sends.clear();
  recvs.clear();
  const int r = L.rank, P = L.nranks;
  for (int q = 0; q < P; ++q) {
    if (dir == A2A_MODE_TO_TIME) {
      for (int i = 0; i < L.ntl[q]; ++i) {  // r -> q: the slices of q's time slab
        const long t = L.t0[q] + i;
        sends.push_back({q, t * L.mode_len[r], 0, L.mode_len[r], i});
      }
      for (int i = 0; i < L.ntl[r]; ++i) {  // q -> r: q's modes of r's slices
        recvs.push_back({q, 0, (long)i * L.npad + L.mode_off[q], L.mode_len[q], i});
      }
    } else {
      for (int i = 0; i < L.ntl[r]; ++i) {  // r -> q: q's modes of r's slices
        sends.push_back({q, (long)i * L.npad + L.mode_off[q], 0, L.mode_len[q], i});
      }
      for (int i = 0; i < L.ntl[q]; ++i) {  // q -> r: r's modes of q's slices
        const long t = L.t0[q] + i;
        recvs.push_back({q, 0, (t + shift) * L.mode_len[r], L.mode_len[r], i});
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// NCCL, loaded at run time
// ---------------------------------------------------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok;
};

static NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the NCCL the process already loaded (torch's), else the default search
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    bool ok = true;
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) ok = false;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = ok;
  });
  return api;
}

static std::string nccl_err(ncclResult_t r) {
  NcclApi& a = nccl();
  return a.ok ? std::string(a.GetErrorString(r)) : std::string("NCCL not loaded");
}

// Execute one schedule (the messages with slice key in [s_lo, s_hi)) through a transport:
// the self part as local copies (the k-th self send paired with the k-th self recv), then
// one group of point-to-point sends and receives in the schedule's order.  Every message's
// slice key is the slice index within the time slab it belongs to, and every rank's slab
// has nt / P slices, so a key range is one symmetric chunk of the all-to-all on every rank.
// The device path runs it with NcclTransport (cudaMemcpyAsync + ncclSend / ncclRecv); the
// CPU tests run the SAME function with a host transport (expd_a2a_execute_host: memcpy +
// the caller's send / recv, torch.distributed gloo in tests/test_dist_cpu.py).
template <class Tr>
static int a2a_run(Tr& tr, const DistLayout& L, const std::vector<A2AMsg>& sends, const std::vector<A2AMsg>& recvs,
                   const double* src, double* dst, std::string& err, int s_lo, int s_hi) {
  auto in = [&](const A2AMsg& m) { return m.slice >= s_lo && m.slice < s_hi; };
  std::vector<const A2AMsg*> ss, rr;
  for (const auto& m : sends)
    if (m.peer == L.rank && in(m)) ss.push_back(&m);
  for (const auto& m : recvs)
    if (m.peer == L.rank && in(m)) rr.push_back(&m);
  if (ss.size() != rr.size()) {
    err = "a2a: self schedule mismatch";
    return EXPD_ERR_INVALID_ARG;
  }
  for (size_t k = 0; k < ss.size(); ++k) {
    if (ss[k]->count != rr[k]->count) {
      err = "a2a: self message sizes differ";
      return EXPD_ERR_INVALID_ARG;
    }
    if (int e = tr.self_copy(dst + rr[k]->dst_off, src + ss[k]->src_off, ss[k]->count, err)) return e;
  }
  if (L.nranks == 1) return EXPD_OK;
  if (int e = tr.group_start(err)) return e;
  int st = EXPD_OK;
  for (const auto& m : sends)
    if (st == EXPD_OK && m.peer != L.rank && in(m)) st = tr.send(src + m.src_off, m.count, m.peer, err);
  for (const auto& m : recvs)
    if (st == EXPD_OK && m.peer != L.rank && in(m)) st = tr.recv(dst + m.dst_off, m.count, m.peer, err);
  const int st2 = tr.group_end(err);  // always close the group
  return st != EXPD_OK ? st : st2;
}

struct NcclTransport {
  void* comm;
  cudaStream_t st;
  int self_copy(double* d, const double* s, long n, std::string& err) {
    cudaError_t e = cudaMemcpyAsync(d, s, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) return EXPD_OK;
    err = std::string("a2a self copy: ") + cudaGetErrorString(e);
    return EXPD_ERR_CUDA;
  }
  int check(ncclResult_t r, std::string& err) {
    if (r == ncclSuccess) return EXPD_OK;
    err = "a2a: " + nccl_err(r);
    return EXPD_ERR_NCCL;
  }
  int group_start(std::string& err) {
    NcclApi& a = nccl();
    if (!a.ok || !comm) {
      err = "a2a: NCCL unavailable";
      return EXPD_ERR_NCCL;
    }
    return check(a.GroupStart(), err);
  }
  int send(const double* b, long n, int peer, std::string& err) {
    return check(nccl().Send(b, (size_t)n, ncclFloat64, peer, (ncclComm_t)comm, st), err);
  }
  int recv(double* b, long n, int peer, std::string& err) {
    return check(nccl().Recv(b, (size_t)n, ncclFloat64, peer, (ncclComm_t)comm, st), err);
  }
  int group_end(std::string& err) {
    NcclApi& a = nccl();
    return a.ok ? check(a.GroupEnd(), err) : EXPD_ERR_NCCL;
  }
};

struct HostTransport {
  const expd_transport* t;
  int self_copy(double* d, const double* s, long n, std::string&) {
    memmove(d, s, sizeof(double) * n);
    return EXPD_OK;
  }
  int wrap(int r, const char* what, std::string& err) {
    if (r == 0) return EXPD_OK;
    err = std::string("a2a host transport: ") + what + " failed";
    return EXPD_ERR_NCCL;
  }
  int group_start(std::string& err) { return wrap(t->group_start ? t->group_start(t->ctx) : 0, "group_start", err); }
  int send(const double* b, long n, int peer, std::string& err) { return wrap(t->send(t->ctx, b, n, peer), "send", err); }
  int recv(double* b, long n, int peer, std::string& err) { return wrap(t->recv(t->ctx, b, n, peer), "recv", err); }
  int group_end(std::string& err) { return wrap(t->group_end ? t->group_end(t->ctx) : 0, "group_end", err); }
};

// ---- host communicators -----------------------------------------------------------------
struct HostComm {
  expd_transport t;
  int rank, nranks;
};
static std::mutex g_hc_mu;
static std::unordered_set<const void*> g_hc;  // live host communicators
static HostComm* host_comm(void* comm) {
  std::lock_guard<std::mutex> lk(g_hc_mu);
  return comm && g_hc.count(comm) ? static_cast<HostComm*>(comm) : nullptr;
}

static int cuda_fail(cudaError_t e, const char* what, std::string& err) {
  if (e == cudaSuccess) return EXPD_OK;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return EXPD_ERR_CUDA;
}

// Device buffers through host staging and a host transport (blocking): group_start waits
// for the stream (the sources are final), each send copies its device range to a host
// buffer and posts it, each receive posts a host buffer, and group_end -- once the transport
// has completed every message -- copies the received buffers to their device ranges.
struct StagedTransport {
  HostComm* hc;
  cudaStream_t st;
  std::vector<std::unique_ptr<double[]>> bufs;  // alive until group_end returns
  std::vector<std::pair<double*, std::pair<const double*, long>>> landing;  // device dst, host src, count
  int self_copy(double* d, const double* s, long n, std::string& err) {
    return cuda_fail(cudaMemcpyAsync(d, s, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "a2a self copy", err);
  }
  int wrap(int r, const char* what, std::string& err) {
    if (r == 0) return EXPD_OK;
    err = std::string("a2a host communicator: ") + what + " failed";
    return EXPD_ERR_NCCL;
  }
  int group_start(std::string& err) {
    bufs.clear();
    landing.clear();
    if (int e = cuda_fail(cudaStreamSynchronize(st), "a2a host communicator", err)) return e;
    return wrap(hc->t.group_start ? hc->t.group_start(hc->t.ctx) : 0, "group_start", err);
  }
  int send(const double* b, long n, int peer, std::string& err) {
    bufs.emplace_back(new double[n > 0 ? n : 1]);
    double* h = bufs.back().get();
    if (int e = cuda_fail(cudaMemcpy(h, b, sizeof(double) * n, cudaMemcpyDeviceToHost), "a2a stage out", err))
      return e;
    return wrap(hc->t.send(hc->t.ctx, h, n, peer), "send", err);
  }
  int recv(double* b, long n, int peer, std::string& err) {
    bufs.emplace_back(new double[n > 0 ? n : 1]);
    double* h = bufs.back().get();
    landing.push_back({b, {h, n}});
    return wrap(hc->t.recv(hc->t.ctx, h, n, peer), "recv", err);
  }
  int group_end(std::string& err) {
    if (int e = wrap(hc->t.group_end ? hc->t.group_end(hc->t.ctx) : 0, "group_end", err)) return e;
    for (const auto& l : landing)
      if (int e = cuda_fail(cudaMemcpyAsync(l.first, l.second.first, sizeof(double) * l.second.second,
                                            cudaMemcpyHostToDevice, st), "a2a stage in", err))
        return e;
    return cuda_fail(cudaStreamSynchronize(st), "a2a stage in", err);  // before bufs are released
  }
};

// Sum over the ranks through a host communicator: every rank sends its count values to
// every other rank and adds the P contributions in rank order, so all ranks hold the same
// bits (as NCCL's allreduce guarantees).
static int host_allreduce(HostComm* hc, double* buf, long count, cudaStream_t st, std::string& err) {
  const int P = hc->nranks, me = hc->rank;
  std::vector<double> all((size_t)P * count);
  if (int e = cuda_fail(cudaMemcpyAsync(all.data() + (size_t)me * count, buf, sizeof(double) * count,
                                        cudaMemcpyDeviceToHost, st), "allreduce stage out", err))
    return e;
  if (int e = cuda_fail(cudaStreamSynchronize(st), "allreduce stage out", err)) return e;
  const expd_transport& t = hc->t;
  if (P > 1) {
    int r = t.group_start ? t.group_start(t.ctx) : 0;
    for (int q = 0; q < P && r == 0; ++q)
      if (q != me) r = t.send(t.ctx, all.data() + (size_t)me * count, count, q);
    for (int q = 0; q < P && r == 0; ++q)
      if (q != me) r = t.recv(t.ctx, all.data() + (size_t)q * count, count, q);
    const int r2 = t.group_end ? t.group_end(t.ctx) : 0;
    if (r || r2) {
      err = "allreduce: host communicator transport failed";
      return EXPD_ERR_NCCL;
    }
  }
  std::vector<double> sum(count, 0.0);
  for (int q = 0; q < P; ++q)
    for (long i = 0; i < count; ++i) sum[i] += all[(size_t)q * count + i];
  if (int e = cuda_fail(cudaMemcpyAsync(buf, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st),
                        "allreduce stage in", err))
    return e;
  return cuda_fail(cudaStreamSynchronize(st), "allreduce stage in", err);
}

int a2a_execute(void* comm, const DistLayout& L, const std::vector<A2AMsg>& sends, const std::vector<A2AMsg>& recvs,
                const double* src, double* dst, cudaStream_t st, std::string& err, int s_lo, int s_hi) {
  if (HostComm* hc = host_comm(comm)) {
    StagedTransport tr{hc, st, {}, {}};
    return a2a_run(tr, L, sends, recvs, src, dst, err, s_lo, s_hi);
  }
  NcclTransport tr{comm, st};
  return a2a_run(tr, L, sends, recvs, src, dst, err, s_lo, s_hi);
}

int allreduce_sum(void* comm, int nranks, double* buf, long count, cudaStream_t st, std::string& err) {
  if (nranks == 1 && !comm) return EXPD_OK;
  if (HostComm* hc = host_comm(comm)) return host_allreduce(hc, buf, count, st, err);
  NcclApi& a = nccl();
  if (!a.ok || !comm) {
    err = "allreduce: NCCL unavailable";
    return EXPD_ERR_NCCL;
  }
  ncclResult_t r = a.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)comm, st);
  if (r != ncclSuccess) {
    err = "allreduce: " + nccl_err(r);
    return EXPD_ERR_NCCL;
  }
  return EXPD_OK;
}

}  // namespace expd

using namespace expd;

// ---------------------------------------------------------------------------------------
// C-ABI (include/expd.h "Multi-GPU")
// ---------------------------------------------------------------------------------------
// the geometry the partition is computed on (complex problems: doubled, as in the plan)
static bool geom_of(const expd_problem* p, Geom* g) {
  if (!p || p->dim < 1 || p->dim > 3 || p->n < 3) return false;
  g->dim = p->dim;
  g->n = p->n;
  g->M = p->n + 1;
  long N = 1, npad = p->n + 1;
  for (int i = 0; i < p->dim; ++i) N *= p->n;
  for (int i = 1; i < p->dim; ++i) npad *= p->n;
  g->N = N;
  g->npad = npad;
  if (p->a_im != 0.0 || p->c_im != 0.0) *g = complex_layout_geom(*g);
  return true;
}

extern "C" expd_status expd_layout_query(const expd_problem* prob, int rank, int nranks, expd_layout* out) {
  Geom g{};
  if (!out || !geom_of(prob, &g)) return EXPD_ERR_INVALID_ARG;
  DistLayout L{};
  if (!dist_layout(g, prob->nt, rank, nranks, &L)) return EXPD_ERR_INVALID_ARG;
  out->rank = rank;
  out->nranks = nranks;
  out->npad = L.npad;
  out->mode_off = L.mode_off[rank];
  out->mode_len = L.mode_len[rank];
  out->t0 = L.t0[rank];
  out->nt_local = L.ntl[rank];
  return EXPD_OK;
}

extern "C" long expd_a2a_schedule(const expd_problem* prob, int rank, int nranks, int direction, int shift,
                                  long* sends, long* recvs, long cap) {
  return expd_a2a_schedule_keyed(prob, rank, nranks, direction, shift, sends, recvs, cap, 4);
}

extern "C" long expd_a2a_schedule_keyed(const expd_problem* prob, int rank, int nranks, int direction, int shift,
                                        long* sends, long* recvs, long cap, int stride) {
  Geom g{};
  if (!geom_of(prob, &g)) return -1;
  DistLayout L{};
  if (!dist_layout(g, prob->nt, rank, nranks, &L)) return -1;
  if (direction != A2A_MODE_TO_TIME && direction != A2A_TIME_TO_MODE) return -1;
  std::vector<A2AMsg> s, r;
  a2a_schedule(L, direction, shift, s, r);
  const long n = (long)s.size();
  if ((long)r.size() != n) return -1;
  if (stride != 4 && stride != 5) return -1;
  if (sends && recvs && cap >= n) {
    for (long i = 0; i < n; ++i) {
      long* o = sends + stride * i;
      long* q = recvs + stride * i;
      o[0] = s[i].peer;
      o[1] = s[i].src_off;
      o[2] = s[i].dst_off;
      o[3] = s[i].count;
      q[0] = r[i].peer;
      q[1] = r[i].src_off;
      q[2] = r[i].dst_off;
      q[3] = r[i].count;
      if (stride == 5) {
        o[4] = s[i].slice;
        q[4] = r[i].slice;
      }
    }
  }
  return n;
}

extern "C" expd_status expd_a2a_execute_host(const expd_problem* prob, int rank, int nranks, int direction,
                                             int shift, int s_lo, int s_hi, const double* src, double* dst,
                                             const expd_transport* transport) {
  Geom g{};
  if (!src || !dst || !transport || !transport->send || !transport->recv || !geom_of(prob, &g))
    return EXPD_ERR_INVALID_ARG;
  DistLayout L{};
  if (!dist_layout(g, prob->nt, rank, nranks, &L)) return EXPD_ERR_INVALID_ARG;
  if (direction != A2A_MODE_TO_TIME && direction != A2A_TIME_TO_MODE) return EXPD_ERR_INVALID_ARG;
  std::vector<A2AMsg> s, r;
  a2a_schedule(L, direction, shift, s, r);
  HostTransport tr{transport};
  std::string err;
  return (expd_status)a2a_run(tr, L, s, r, src, dst, err, s_lo, s_hi);
}

extern "C" expd_status expd_nccl_unique_id(unsigned char id[128]) {
  NcclApi& a = nccl();
  if (!id) return EXPD_ERR_INVALID_ARG;
  if (!a.ok) return EXPD_ERR_NCCL;
  ncclUniqueId u;
  if (a.GetUniqueId(&u) != ncclSuccess) return EXPD_ERR_NCCL;
  static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
  memcpy(id, u.internal, 128);
  return EXPD_OK;
}

extern "C" expd_status expd_nccl_comm_init(const unsigned char id[128], int nranks, int rank, int device,
                                           void** comm) {
  NcclApi& a = nccl();
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return EXPD_ERR_INVALID_ARG;
  if (!a.ok) return EXPD_ERR_NCCL;
  if (cudaSetDevice(device) != cudaSuccess) return EXPD_ERR_CUDA;
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  if (a.CommInitRank(&c, nranks, u, rank) != ncclSuccess) return EXPD_ERR_NCCL;
  *comm = (void*)c;
  return EXPD_OK;
}

extern "C" void expd_nccl_comm_destroy(void* comm) {
  if (host_comm(comm)) return;  // not an NCCL communicator (expd_host_comm_destroy owns it)
  NcclApi& a = nccl();
  if (comm && a.ok) a.CommDestroy((ncclComm_t)comm);
}

extern "C" expd_status expd_host_comm_create(const expd_transport* transport, int rank, int nranks, void** comm) {
  if (!transport || !transport->send || !transport->recv || !comm || nranks < 1 || rank < 0 || rank >= nranks)
    return EXPD_ERR_INVALID_ARG;
  HostComm* hc = new HostComm{*transport, rank, nranks};
  std::lock_guard<std::mutex> lk(g_hc_mu);
  g_hc.insert(hc);
  *comm = hc;
  return EXPD_OK;
}

extern "C" void expd_host_comm_destroy(void* comm) {
  std::lock_guard<std::mutex> lk(g_hc_mu);
  if (comm && g_hc.erase(comm)) delete static_cast<HostComm*>(comm);
}
