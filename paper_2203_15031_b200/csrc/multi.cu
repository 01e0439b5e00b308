// Multi-device host entry (spmesl_fit / spmesl_fit_ex with options.num_devices >= 1): one
// process drives G devices of one node with NCCL (BASELINE.json north_star (3); SURVEY.md §8(e);
// DESIGN.md §8).  The p column problems are independent, so each device fits a
// contiguous column block with X replicated; the exchanges are
//   1. the first-sweep screening flags: every device screens an equal share of the screening
//      tiles, then one max all-reduce of p bytes (the flags of all pairs);
//   2. after the fit, one all-gather of the fitted coefficients as CSC (per-column counts,
//      sigma, rows and values: the nonzeros, not p x p doubles);
// after which device 0 symmetrizes (Eq. symm, P:388-394 — it needs b_kj from column j's owner)
// and assembles Theta as COO entries + diagonal, which the host scatters into the caller's
// dense Theta (zero-filled by host threads meanwhile, as in the single-device path).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy the process already has —
// e.g. torch's — else the system's, else the pip package's): the library links and loads without
// it, and a multi-device call without it returns SPMESL_ERR_NCCL.  One host thread per device
// runs its building blocks (the C entry points of spmesl.h on that device) and its collectives;
// the threads meet at a rendezvous before every collective so that an error on any device is
// seen by all of them (no device enters a collective its peers will not join).
#include <dlfcn.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nccl.h>

#include "spmesl.h"
#include "spmesl_internal.cuh"

namespace spmesl {

int multi_fail(int code, const std::string& msg);   // (api.cu: sets spmesl_last_error)

namespace {

struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;

#ifndef SPMESL_NCCL_PIP_LIB
#define SPMESL_NCCL_PIP_LIB ""
#endif

const NcclApi& nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h && SPMESL_NCCL_PIP_LIB[0]) h = dlopen(SPMESL_NCCL_PIP_LIB, RTLD_NOW);
  if (!h) { g_nccl.why = "libnccl.so.2 not found"; return g_nccl; }
  g_nccl.CommInitAll = (decltype(&ncclCommInitAll))dlsym(h, "ncclCommInitAll");
  g_nccl.CommDestroy = (decltype(&ncclCommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(&ncclAllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.AllGather = (decltype(&ncclAllGather))dlsym(h, "ncclAllGather");
  g_nccl.GetErrorString = (decltype(&ncclGetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.CommInitAll && g_nccl.CommDestroy && g_nccl.AllReduce && g_nccl.AllGather &&
              g_nccl.GetErrorString;
  if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks a required symbol";
  return g_nccl;
}

// communicators for one device list, created once (ncclCommInitAll) and kept
struct CommSet {
  std::vector<int> devs;
  std::vector<ncclComm_t> comms;
};
std::mutex g_comm_mu;
std::vector<CommSet*> g_comm_sets;

int comms_for(const std::vector<int>& devs, CommSet** out) {
  const NcclApi& A = nccl_api();
  if (!A.ok) return multi_fail(SPMESL_ERR_NCCL, "NCCL unavailable: " + A.why);
  std::lock_guard<std::mutex> lk(g_comm_mu);
  for (CommSet* c : g_comm_sets)
    if (c->devs == devs) { *out = c; return SPMESL_OK; }
  CommSet* c = new CommSet();
  c->devs = devs;
  c->comms.resize(devs.size());
  const ncclResult_t r = A.CommInitAll(c->comms.data(), (int)devs.size(), devs.data());
  if (r != ncclSuccess) {
    delete c;
    return multi_fail(SPMESL_ERR_NCCL, std::string("ncclCommInitAll: ") + A.GetErrorString(r));
  }
  g_comm_sets.push_back(c);
  *out = c;
  return SPMESL_OK;
}

// all device threads meet here; the first nonzero code any of them brought is returned to all
struct Rendezvous {
  std::mutex mu;
  std::condition_variable cv;
  int n, arrived = 0, gen = 0, code = 0;
  std::string msg;
  explicit Rendezvous(int n_) : n(n_) {}
  int meet(int code_in, const std::string& msg_in) {
    std::unique_lock<std::mutex> lk(mu);
    if (code_in < 0 && code == 0) { code = code_in; msg = msg_in; }
    const int g = gen;
    if (++arrived == n) { arrived = 0; ++gen; cv.notify_all(); }
    else cv.wait(lk, [&] { return gen != g; });
    return code;
  }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  }
};

void column_range(int64_t p, int rank, int world, int64_t* c0, int64_t* c1) {
  const int64_t base = p / world, rem = p % world;
  *c0 = rank * base + std::min<int64_t>(rank, rem);
  *c1 = *c0 + base + (rank < rem ? 1 : 0);
}

}  // namespace

// The multi-device fit of spmesl_fit_ex (host X, host outputs).  o.num_devices >= 1.
int fit_multi_device(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                     int32_t max_iter, const spmesl_options& o, double* Theta, double* sigma,
                     int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st) {
  const int G = o.num_devices;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) { cudaGetLastError(); ndev = 0; }
  std::vector<int> devs(G);
  for (int d = 0; d < G; ++d) devs[d] = o.device_ids ? o.device_ids[d] : d;
  bool dup = false;
  for (int d = 0; d < G; ++d) {
    if (devs[d] < 0 || devs[d] >= ndev)
      return multi_fail(SPMESL_ERR_ARG, "device id " + std::to_string(devs[d]) + " is not a device");
    for (int e = 0; e < d; ++e) dup = dup || devs[e] == devs[d];
  }
  if (G > p) return multi_fail(SPMESL_ERR_ARG, "more devices than columns");
  if (o.mode != 0)
    return multi_fail(SPMESL_ERR_UNSUPPORTED, "mode 1 (joint stop over all columns) runs on one device");
  if (o.exchange < 0 || o.exchange > 2) return multi_fail(SPMESL_ERR_ARG, "bad options.exchange");
  // exchange: peer-to-peer when every pair of distinct devices has peer access (NVLink /
  // NVSwitch), else NCCL collectives (options.exchange forces one)
  bool peer_ok = G <= kP2PMax;
  for (int d = 0; d < G && peer_ok; ++d)
    for (int e = 0; e < G && peer_ok; ++e) {
      if (devs[e] == devs[d]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, devs[d], devs[e]) != cudaSuccess) { cudaGetLastError(); can = 0; }
      peer_ok = can != 0;
    }
  const bool p2p = o.exchange == 2 || (o.exchange == 0 && peer_ok);
  if (p2p && !peer_ok)
    return multi_fail(SPMESL_ERR_UNSUPPORTED, G > kP2PMax ? "peer-to-peer exchange: at most 16 devices"
                                                          : "peer-to-peer exchange: no peer access between two of the devices");
  if (dup && !p2p)
    return multi_fail(SPMESL_ERR_ARG, "device ids must be distinct (NCCL exchange)");
  CommSet* cs = nullptr;
  int rc = p2p ? SPMESL_OK : comms_for(devs, &cs);
  if (rc) return rc;
  const NcclApi& A = nccl_api();
  const size_t pp = (size_t)p * (size_t)p;
  // the caller's dense Theta is zero-filled by host threads while the devices compute
  std::vector<std::thread> zero;
  {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const size_t nth = std::min<size_t>(std::min(16u, hc), std::max<size_t>(1, pp >> 20));
    const size_t per = (pp + nth - 1) / nth;
    for (size_t t = 0; t < nth; ++t) {
      const size_t lo = t * per, hi = std::min(pp, lo + per);
      if (lo < hi) zero.emplace_back([=] { std::memset(Theta + lo, 0, (hi - lo) * sizeof(double)); });
    }
  }
  spmesl_options od = o;
  od.num_devices = 0;      // the building blocks run on the current device
  od.device_ids = nullptr;
  od.device = -1;
  const bool gram = spmesl_gram_supported(n, p) != 0 && o.solver != 1;
  const int64_t m_max = (p + G - 1) / G;
  Rendezvous rv(G);
  std::vector<int64_t> nnz(G, 0);
  std::vector<spmesl_stats> dst(G);
  std::vector<int> rcs(G, 0);
  // device 0's results for the host
  std::vector<int32_t> cr, cc;
  std::vector<double> cv, diag((size_t)p);
  double ms_comm = 0.0;
  // peer-to-peer exchange: every device's published buffers, and its symmetrized entries
  P2PBlocks pb;
  std::memset(&pb, 0, sizeof(pb));
  pb.p = p;
  pb.G = G;
  std::vector<std::vector<int32_t>> pcr(G), pcc(G);
  std::vector<std::vector<double>> pcv(G);
  auto worker = [&](int d) {
    int code = 0;
    std::string msg;
    auto err = [&](int c, const std::string& m) { if (!code) { code = c; msg = m; } };
#define MTRY(expr)                                                                     \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) err(e_ == cudaErrorMemoryAllocation ? SPMESL_ERR_OOM : SPMESL_ERR_CUDA, \
                               std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)
#define NTRY(expr)                                                                     \
  do {                                                                                 \
    ncclResult_t r_ = (expr);                                                          \
    if (r_ != ncclSuccess) err(SPMESL_ERR_NCCL, std::string(#expr) + ": " + A.GetErrorString(r_)); \
  } while (0)
    MTRY(cudaSetDevice(devs[d]));
    if (p2p)
      for (int e = 0; e < G; ++e) {
        bool seen = devs[e] == devs[d];
        for (int f = 0; f < e && !seen; ++f) seen = devs[f] == devs[e];
        if (seen) continue;
        const cudaError_t pe = cudaDeviceEnablePeerAccess(devs[e], 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else MTRY(pe);
      }
    cudaStream_t s = nullptr;
    MTRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
    MTRY(cudaEventCreate(&e0)); MTRY(cudaEventCreate(&e1));
    MTRY(cudaEventCreate(&e2)); MTRY(cudaEventCreate(&e3));
    int64_t c0, c1;
    column_range(p, d, G, &c0, &c1);
    const int64_t m = c1 - c0;
    DevBuf<double> dX, sig, scale, sig_all, vals, vals_all;
    DevBuf<uint8_t> hit, share, conv;
    DevBuf<int64_t> cpb, cpt;              // (p2p) this block's CSC column pointers
    DevBuf<int32_t> crow, ccol;            // (p2p) this block's symmetrized entries
    DevBuf<double> cvals, dgb, sgb;
    DevBuf<int> ccount;
    DevBuf<int32_t> cnt, cnt_all, rows, rows_all, it, sw;
    MTRY(dX.alloc((size_t)n * p)); MTRY(hit.alloc(p)); MTRY(sig.alloc(m_max));
    MTRY(scale.alloc(p)); MTRY(cnt.alloc(m_max)); MTRY(it.alloc(m)); MTRY(sw.alloc(m));
    MTRY(conv.alloc(m));
    if (!code) {
      MTRY(cudaMemcpyAsync(dX.p, X, (size_t)n * p * 8, cudaMemcpyHostToDevice, s));
      MTRY(cudaMemsetAsync(hit.p, 0, p, s));
      if (p2p) { MTRY(share.alloc(p)); if (!code) MTRY(cudaMemsetAsync(share.p, 0, p, s)); }
      MTRY(cudaMemsetAsync(cnt.p, 0, (size_t)m_max * 4, s));
      MTRY(cudaMemsetAsync(sig.p, 0, (size_t)m_max * 8, s));
    }
    // (1) screening share + flag all-reduce (Gram solver)
    if (!code && gram) {
      const int64_t nt = spmesl_screen_tile_count(p, &od);
      int64_t t0, t1;
      column_range(nt, d, G, &t0, &t1);
      spmesl_stats ss;
      const int r = spmesl_gram_screen_device(dX.p, n, p, lambda0, t0, t1, &od,
                                              p2p ? share.p : hit.p, s, &ss);
      if (r < 0) err(r, spmesl_last_error());
      pb.flags[d] = share.p;
    }
    code = rv.meet(code, msg);
    if (!code && gram && p2p) {   // flags of every share, read from the peers' memory
      MTRY(cudaEventRecord(e0, s));
      MTRY(launch_p2p_flag_max(pb, hit.p, s));
      MTRY(cudaEventRecord(e1, s));
      MTRY(cudaStreamSynchronize(s));
    }
    if (!code && gram && !p2p) {
      MTRY(cudaEventRecord(e0, s));
      NTRY(A.AllReduce(hit.p, hit.p, (size_t)p, ncclUint8, ncclMax, cs->comms[d], s));
      MTRY(cudaEventRecord(e1, s));
      MTRY(cudaStreamSynchronize(s));
    }
    // (2) this device's column block, exported as CSC (retried once with the capacity needed)
    if (!code) {
      int64_t cap = std::max<int64_t>(m * 16, 1024);
      for (int attempt = 0; attempt < 2 && !code; ++attempt) {
        MTRY(rows.alloc(cap)); MTRY(vals.alloc(cap));
        if (code) break;
        int64_t nz = 0;
        int r;
        if (gram)
          r = spmesl_fit_columns_gram_device(dX.p, n, p, c0, c1, lambda0, tol, max_iter, &od, hit.p,
                                             cnt.p, rows.p, vals.p, cap, &nz, sig.p, scale.p, it.p,
                                             sw.p, conv.p, s, &dst[d]);
        else
          r = spmesl_fit_columns_device(dX.p, n, p, c0, c1, lambda0, tol, max_iter, &od, cnt.p,
                                        rows.p, vals.p, cap, &nz, sig.p, scale.p, it.p, sw.p,
                                        conv.p, s, &dst[d]);
        if (r == SPMESL_ERR_ARG && nz > cap) { cap = nz; continue; }
        if (r < 0) err(r, spmesl_last_error());
        rcs[d] = r;
        nnz[d] = nz;
        break;
      }
    }
    if (!code) {   // per-column results of this block straight to the caller
      MTRY(cudaMemcpyAsync(iters + c0, it.p, (size_t)m * 4, cudaMemcpyDeviceToHost, s));
      if (sweeps) MTRY(cudaMemcpyAsync(sweeps + c0, sw.p, (size_t)m * 4, cudaMemcpyDeviceToHost, s));
      if (converged) MTRY(cudaMemcpyAsync(converged + c0, conv.p, (size_t)m, cudaMemcpyDeviceToHost, s));
      MTRY(cudaStreamSynchronize(s));
    }
    if (p2p) {
      // publish this block's CSC for the peers, meet, and symmetrize the own columns by
      // reading each partner b_kj (and sigma_j) on the device that owns column j
      if (!code) {
        MTRY(cpb.alloc(m + 1)); MTRY(cpt.alloc(1));
        if (!code) MTRY(launch_csc_scan(cnt.p, (int)m, cpb.p, cpt.p, s));
        MTRY(cudaStreamSynchronize(s));
        pb.col_ptr[d] = cpb.p; pb.rows[d] = rows.p; pb.vals[d] = vals.p; pb.sigma_std[d] = sig.p;
        MTRY(crow.alloc(nnz[d])); MTRY(ccol.alloc(nnz[d])); MTRY(cvals.alloc(nnz[d]));
        MTRY(dgb.alloc(m)); MTRY(sgb.alloc(m)); MTRY(ccount.alloc(1));
      }
      code = rv.meet(code, msg);
      if (!code) {
        MTRY(cudaEventRecord(e2, s));
        MTRY(launch_assemble_coo_p2p(pb, d, o.standardize ? scale.p : nullptr, o.symmetrize, crow.p,
                                     ccol.p, cvals.p, ccount.p, dgb.p, sgb.p, s));
        MTRY(cudaEventRecord(e3, s));
        int ncoo = 0;
        MTRY(cudaMemcpyAsync(&ncoo, ccount.p, 4, cudaMemcpyDeviceToHost, s));
        MTRY(cudaStreamSynchronize(s));
        if (!code) {
          pcr[d].resize(ncoo); pcc[d].resize(ncoo); pcv[d].resize(ncoo);
          if (ncoo) {
            MTRY(cudaMemcpyAsync(pcr[d].data(), crow.p, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
            MTRY(cudaMemcpyAsync(pcc[d].data(), ccol.p, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
            MTRY(cudaMemcpyAsync(pcv[d].data(), cvals.p, (size_t)ncoo * 8, cudaMemcpyDeviceToHost, s));
          }
          MTRY(cudaMemcpyAsync(diag.data() + c0, dgb.p, (size_t)m * 8, cudaMemcpyDeviceToHost, s));
          MTRY(cudaMemcpyAsync(sigma + c0, sgb.p, (size_t)m * 8, cudaMemcpyDeviceToHost, s));
          MTRY(cudaStreamSynchronize(s));
        }
        if (!code && d == 0) {
          float a = 0.f, b = 0.f;
          if (gram && cudaEventElapsedTime(&a, e0, e1) != cudaSuccess) { cudaGetLastError(); a = 0.f; }
          if (cudaEventElapsedTime(&b, e2, e3) != cudaSuccess) { cudaGetLastError(); b = 0.f; }
          ms_comm = (double)a + (double)b;
        }
      }
      // no device frees its buffers while a peer may still read them
      code = rv.meet(code, msg);
    }
    if (!p2p) code = rv.meet(code, msg);   // (every nnz[] is known past this point)
    int64_t nnz_max = 1;
    for (int e = 0; e < G; ++e) nnz_max = std::max(nnz_max, nnz[e]);
    // (3) all-gather of the CSC blocks (padded to the largest block)
    if (!code && !p2p) {
      MTRY(cnt_all.alloc((size_t)G * m_max)); MTRY(sig_all.alloc((size_t)G * m_max));
      MTRY(rows_all.alloc((size_t)G * nnz_max)); MTRY(vals_all.alloc((size_t)G * nnz_max));
      if (nnz_max > nnz[d] && rows.p) {   // (grow this block's buffers to the padded size)
        DevBuf<int32_t> r2; DevBuf<double> v2;
        MTRY(r2.alloc(nnz_max)); MTRY(v2.alloc(nnz_max));
        if (!code) {
          MTRY(cudaMemcpyAsync(r2.p, rows.p, (size_t)nnz[d] * 4, cudaMemcpyDeviceToDevice, s));
          MTRY(cudaMemcpyAsync(v2.p, vals.p, (size_t)nnz[d] * 8, cudaMemcpyDeviceToDevice, s));
          std::swap(rows.p, r2.p);
          std::swap(vals.p, v2.p);
        }
      }
    }
    if (!p2p) code = rv.meet(code, msg);
    if (!code && !p2p) {
      MTRY(cudaEventRecord(e2, s));
      NTRY(A.AllGather(cnt.p, cnt_all.p, (size_t)m_max, ncclInt32, cs->comms[d], s));
      NTRY(A.AllGather(sig.p, sig_all.p, (size_t)m_max, ncclFloat64, cs->comms[d], s));
      NTRY(A.AllGather(rows.p, rows_all.p, (size_t)nnz_max, ncclInt32, cs->comms[d], s));
      NTRY(A.AllGather(vals.p, vals_all.p, (size_t)nnz_max, ncclFloat64, cs->comms[d], s));
      MTRY(cudaEventRecord(e3, s));
      MTRY(cudaStreamSynchronize(s));
    }
    // (4) device 0: the global CSC (ranks in column order), symmetrized COO + diagonal
    if (!code && d == 0 && !p2p) {
      DevBuf<int32_t> cnt_g, rows_g;
      DevBuf<double> sig_g, vals_g, cvals, dg, sg;
      DevBuf<int64_t> col_ptr, total;
      DevBuf<int32_t> crow, ccol;
      DevBuf<int> ccount;
      int64_t tot = 0;
      for (int e = 0; e < G; ++e) tot += nnz[e];
      MTRY(cnt_g.alloc(p)); MTRY(sig_g.alloc(p)); MTRY(rows_g.alloc(tot)); MTRY(vals_g.alloc(tot));
      MTRY(col_ptr.alloc(p + 1)); MTRY(total.alloc(1)); MTRY(crow.alloc(tot)); MTRY(ccol.alloc(tot));
      MTRY(cvals.alloc(tot)); MTRY(dg.alloc(p)); MTRY(sg.alloc(p)); MTRY(ccount.alloc(1));
      int64_t off = 0;
      for (int e = 0; e < G && !code; ++e) {
        int64_t b0, b1;
        column_range(p, e, G, &b0, &b1);
        MTRY(cudaMemcpyAsync(cnt_g.p + b0, cnt_all.p + (size_t)e * m_max, (size_t)(b1 - b0) * 4,
                             cudaMemcpyDeviceToDevice, s));
        MTRY(cudaMemcpyAsync(sig_g.p + b0, sig_all.p + (size_t)e * m_max, (size_t)(b1 - b0) * 8,
                             cudaMemcpyDeviceToDevice, s));
        if (nnz[e]) {
          MTRY(cudaMemcpyAsync(rows_g.p + off, rows_all.p + (size_t)e * nnz_max, (size_t)nnz[e] * 4,
                               cudaMemcpyDeviceToDevice, s));
          MTRY(cudaMemcpyAsync(vals_g.p + off, vals_all.p + (size_t)e * nnz_max, (size_t)nnz[e] * 8,
                               cudaMemcpyDeviceToDevice, s));
        }
        off += nnz[e];
      }
      if (!code) {
        MTRY(launch_csc_scan(cnt_g.p, (int)p, col_ptr.p, total.p, s));
        MTRY(launch_assemble_coo(p, col_ptr.p, rows_g.p, vals_g.p, sig_g.p,
                                 o.standardize ? scale.p : nullptr, o.symmetrize, crow.p, ccol.p,
                                 cvals.p, ccount.p, dg.p, sg.p, s));
        int ncoo = 0;
        MTRY(cudaMemcpyAsync(&ncoo, ccount.p, 4, cudaMemcpyDeviceToHost, s));
        MTRY(cudaStreamSynchronize(s));
        if (!code) {
          cr.resize(ncoo); cc.resize(ncoo); cv.resize(ncoo);
          if (ncoo) {
            MTRY(cudaMemcpyAsync(cr.data(), crow.p, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
            MTRY(cudaMemcpyAsync(cc.data(), ccol.p, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
            MTRY(cudaMemcpyAsync(cv.data(), cvals.p, (size_t)ncoo * 8, cudaMemcpyDeviceToHost, s));
          }
          MTRY(cudaMemcpyAsync(diag.data(), dg.p, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
          MTRY(cudaMemcpyAsync(sigma, sg.p, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
          MTRY(cudaStreamSynchronize(s));
        }
      }
      if (!code) {
        float a = 0.f, b = 0.f;
        if (gram && cudaEventElapsedTime(&a, e0, e1) != cudaSuccess) { cudaGetLastError(); a = 0.f; }
        if (cudaEventElapsedTime(&b, e2, e3) != cudaSuccess) { cudaGetLastError(); b = 0.f; }
        ms_comm = (double)a + (double)b;
      }
    }
    if (code) rcs[d] = code;
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (e2) cudaEventDestroy(e2);
    if (e3) cudaEventDestroy(e3);
    if (s) cudaStreamDestroy(s);
    if (code) { std::lock_guard<std::mutex> lk(rv.mu); if (!rv.code) { rv.code = code; rv.msg = msg; } }
#undef MTRY
#undef NTRY
  };
  int prev = -1;
  cudaGetDevice(&prev);
  std::vector<std::thread> th;
  for (int d = 0; d < G; ++d) th.emplace_back(worker, d);
  for (auto& t : th) t.join();
  for (auto& t : zero) t.join();
  if (prev >= 0) cudaSetDevice(prev);
  if (rv.code) return multi_fail(rv.code, rv.msg);
  for (size_t e = 0; e < cr.size(); ++e) Theta[(size_t)cc[e] * p + cr[e]] = cv[e];
  for (int d = 0; d < G; ++d)
    for (size_t e = 0; e < pcr[d].size(); ++e) Theta[(size_t)pcc[d][e] * p + pcr[d][e]] = pcv[d][e];
  for (int64_t k = 0; k < p; ++k) Theta[(size_t)k * p + k] = diag[k];
  int worst = SPMESL_OK;
  for (int d = 0; d < G; ++d) worst = std::max(worst, rcs[d]);
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->bad_column = -1;
    for (int d = 0; d < G; ++d) {
      st->coord_updates += dst[d].coord_updates;
      st->total_sweeps += dst[d].total_sweeps;
      st->max_sweeps = std::max(st->max_sweeps, dst[d].max_sweeps);
      st->max_outer = std::max(st->max_outer, dst[d].max_outer);
      st->n_unconverged += dst[d].n_unconverged;
      st->kernel_launches += dst[d].kernel_launches;
      st->nnz += dst[d].nnz;
      st->tail_columns += dst[d].tail_columns;
      st->tail_sweeps += dst[d].tail_sweeps;
      st->ms_total = std::max(st->ms_total, dst[d].ms_total);
    }
    st->solver = dst[0].solver;
    st->ms_comm = ms_comm;
    st->num_devices = G;
    st->exchange = p2p ? 2 : 1;
  }
  return worst;
}

}  // namespace spmesl
