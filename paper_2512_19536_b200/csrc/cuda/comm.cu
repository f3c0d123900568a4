// Multi-GPU plumbing: one process per GPU, NCCL over NVLink/NVSwitch.
//
// Subdomains are sharded over ranks as contiguous internal cell ranges
// (host/problem.cpp), so the data path needs exactly three exchanges per PCG
// iteration: the p-halo before the SpMV (grouped
// ncclSend/ncclRecv), scalar all-reduces for the dot products, and an
// all-reduce of the coarse residual r0 (each rank then solves K0 redundantly).
// NCCL is loaded with dlopen so the single-GPU library has no link-time
// dependency; inside a torch process the already-loaded libnccl is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstring>
#include <string>

#include "../host/problem.hpp"
#include "sim.cuh"

namespace pdg {

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.handle) return api;
  const char* names[] = {"libnccl.so.2", "libnccl.so", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
  for (const char* n : names) {
    api.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (api.handle) break;
  }
  if (!api.handle) throw CudaError("NCCL is not available (dlopen libnccl.so.2 failed)");
  auto sym = [](const char* s) {
    void* p = dlsym(nccl().handle, s);
    if (!p) throw CudaError(std::string("NCCL symbol missing: ") + s);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}

template <class T>
T* dmalloc(std::size_t n) {
  T* p = nullptr;
  PDG_CUDA(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)));
  return p;
}

}  // namespace

// ---- transports ----
// NCCL: one communicator per rank (one process per GPU), stream-ordered.
class NcclTransport final : public Transport {
 public:
  explicit NcclTransport(ncclComm_t c) : comm_(c) {}
  ~NcclTransport() override { nccl().CommDestroy(comm_); }
  void allreduce(const double* src, double* dst, long long count, cudaStream_t st) override {
    nccl_check(nccl().AllReduce(src, dst, static_cast<size_t>(count), ncclFloat64, ncclSum, comm_, st),
               "ncclAllReduce");
  }
  void exchange(DeviceSim& s, double* v, cudaStream_t st) override {
    auto& api = nccl();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const auto& h : s.halo_peers) {
      if (h.send_count)
        nccl_check(api.Send(s.d_sendbuf + static_cast<long long>(h.send_off) * s.b,
                            static_cast<size_t>(h.send_count) * s.b, ncclFloat64, h.peer, comm_, st),
                   "ncclSend");
      if (h.recv_count)
        nccl_check(api.Recv(v + (static_cast<long long>(s.ncells) + h.recv_off) * s.b,
                            static_cast<size_t>(h.recv_count) * s.b, ncclFloat64, h.peer, comm_, st),
                   "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_;
};

// Loopback: `world` DeviceSims in ONE process (any devices, typically one
// GPU), each driven by its own host thread. Every exchange goes through host
// staging between two barriers: a test transport that runs the complete
// multi-rank data path (halo pack, halo tail layout, combined coarse/dot
// all-reduce, finish kernels, redundant coarse solve, host-driven loop) where
// NCCL cannot (it rejects two ranks on one device). Sums run in rank order.
struct LoopbackGroup {
  explicit LoopbackGroup(int w) : world(w), buf(w), peers(w, nullptr), sims(w, nullptr) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<double>> buf;           // per rank staging
  std::vector<const std::vector<DeviceSim::HaloPeer>*> peers;
  std::vector<DeviceSim*> sims;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen; }))
      throw CudaError("loopback transport: a peer rank did not arrive (timeout)");
  }
};

class LoopbackTransport final : public Transport {
 public:
  LoopbackTransport(std::shared_ptr<LoopbackGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  void allreduce(const double* src, double* dst, long long count, cudaStream_t st) override {
    auto& mine = g_->buf[rank_];
    mine.resize(static_cast<std::size_t>(count));
    PDG_CUDA(cudaMemcpyAsync(mine.data(), src, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
    sum_.assign(static_cast<std::size_t>(count), 0.0);
    for (int r = 0; r < g_->world; ++r) {
      if (static_cast<long long>(g_->buf[r].size()) != count)
        throw CudaError("loopback transport: all-reduce sizes differ between ranks");
      for (long long i = 0; i < count; ++i) sum_[i] += g_->buf[r][i];
    }
    g_->barrier();  // every rank has read every buffer
    PDG_CUDA(cudaMemcpyAsync(dst, sum_.data(), count * sizeof(double), cudaMemcpyHostToDevice, st));
    PDG_CUDA(cudaStreamSynchronize(st));
  }
  void exchange(DeviceSim& s, double* v, cudaStream_t st) override {
    long long nsend = 0;
    for (const auto& h : s.halo_peers) nsend = std::max<long long>(nsend, h.send_off + h.send_count);
    auto& mine = g_->buf[rank_];
    mine.resize(static_cast<std::size_t>(nsend * s.b));
    if (nsend)
      PDG_CUDA(cudaMemcpyAsync(mine.data(), s.d_sendbuf, nsend * s.b * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    g_->peers[rank_] = &s.halo_peers;
    g_->barrier();
    for (const auto& h : s.halo_peers) {
      if (!h.recv_count) continue;
      const DeviceSim::HaloPeer* src = nullptr;
      for (const auto& o : *g_->peers[h.peer])
        if (o.peer == rank_) src = &o;
      if (!src || src->send_count != h.recv_count)
        throw CudaError("loopback transport: halo plans of the two ranks disagree");
      PDG_CUDA(cudaMemcpyAsync(v + (static_cast<long long>(s.ncells) + h.recv_off) * s.b,
                               g_->buf[h.peer].data() + static_cast<long long>(src->send_off) * s.b,
                               static_cast<std::size_t>(h.recv_count) * s.b * sizeof(double), cudaMemcpyHostToDevice,
                               st));
    }
    PDG_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
  }
  const char* name() const override { return "loopback"; }

 private:
  std::shared_ptr<LoopbackGroup> g_;
  int rank_;
  std::vector<double> sum_;
};

void DeviceSim::comm_allreduce(const double* src, double* dst, long long count) {
  transport->allreduce(src, dst, count, st);
}

void DeviceSim::comm_exchange(double* v, cudaStream_t on) { transport->exchange(*this, v, on); }

void DeviceSim::spmv_overlapped(double* v, double* y) {
  for (const HaloPeer& h : halo_peers)
    launch_pack(v, d_send_cells + h.send_off, h.send_count, b, d_sendbuf + static_cast<long long>(h.send_off) * b, st);
  PDG_CUDA(cudaEventRecord(ev_pack, st));
  // p.q partial: interior rows store it, the halo rows add theirs (fixed order)
  launch_spmv(b, n_rows_int, d_ptr, d_col, d_kval, v, y, v, rctx(kFinStore, d_dot_local), true, st, d_rows_int);
  PDG_CUDA(cudaStreamWaitEvent(st_comm, ev_pack, 0));
  comm_exchange(v, st_comm);
  PDG_CUDA(cudaEventRecord(ev_halo, st_comm));
  PDG_CUDA(cudaStreamWaitEvent(st, ev_halo, 0));
  launch_spmv(b, n_rows_bnd, d_ptr, d_col, d_kval, v, y, v, rctx(n_rows_int > 0 ? kFinAccum : kFinStore, d_dot_local),
              true, st, d_rows_bnd);
}

void DeviceSim::comm_destroy() { transport.reset(); }

void DeviceSim::attach_comm(const void* id128, int r, int w) {
  Problem& pr = *P;
  if (w != pr.cfg.world || r != pr.cfg.rank)
    throw ConfigError("attach_comm: rank/world differ from the configuration the problem was built for");
  if (w == 1) return;
  // K0 below is all-reduced in place: a second attach would scale it by world
  if (transport) throw ConfigError("attach_comm: a communicator is already attached");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  PDG_CUDA(cudaSetDevice(pr.cfg.device));
  nccl_check(nccl().CommInitRank(&c, w, id, r), "ncclCommInitRank");
  connect(std::make_unique<NcclTransport>(c));
}

void DeviceSim::attach_loopback(const std::shared_ptr<LoopbackGroup>& g, int r, int w) {
  Problem& pr = *P;
  if (w != pr.cfg.world || r != pr.cfg.rank || w != g->world)
    throw ConfigError("attach_loopback: rank/world differ from the configuration the problem was built for");
  if (w == 1) return;
  if (transport) throw ConfigError("attach_comm: a communicator is already attached");
  PDG_CUDA(cudaSetDevice(pr.cfg.device));
  connect(std::make_unique<LoopbackTransport>(g, r));
}

// halo plan, reduction scratch, K0 summed over ranks, coarse factor
void DeviceSim::connect(std::unique_ptr<Transport> t) {
  Problem& pr = *P;
  const int r = pr.cfg.rank, w = pr.cfg.world;
  transport = std::move(t);
  d_dot_local = dmalloc<double>(1);
  d_dot_global = dmalloc<double>(1);

  // halo plan from the global mesh adjacency (identical on every rank, host/pack.cpp)
  std::vector<std::vector<int>> send, recv;
  halo_plan(pr, send, recv);
  std::vector<int> send_cells;
  halo_peers.clear();
  for (int peer = 0; peer < w; ++peer) {
    if (peer == r) continue;
    const auto& sc = send[peer];
    HaloPeer h{peer, static_cast<int>(send_cells.size()), static_cast<int>(sc.size()), 0, 0};
    send_cells.insert(send_cells.end(), sc.begin(), sc.end());
    const auto lo = std::lower_bound(halo_cells.begin(), halo_cells.end(), pr.rank_cell_start[peer]);
    const auto hi = std::lower_bound(halo_cells.begin(), halo_cells.end(), pr.rank_cell_start[peer + 1]);
    h.recv_off = static_cast<int>(lo - halo_cells.begin());
    h.recv_count = static_cast<int>(hi - lo);
    if (h.recv_count != static_cast<int>(recv[peer].size()) ||
        !std::equal(recv[peer].begin(), recv[peer].end(), lo))
      throw CudaError("attach_comm: halo plan disagrees with the operator's column set");
    if (h.send_count || h.recv_count) halo_peers.push_back(h);
  }
  d_send_cells = dmalloc<int>(send_cells.size());
  if (!send_cells.empty())
    PDG_CUDA(cudaMemcpy(d_send_cells, send_cells.data(), send_cells.size() * sizeof(int), cudaMemcpyHostToDevice));
  d_sendbuf = dmalloc<double>(send_cells.size() * static_cast<std::size_t>(b));
  // rows that read no halo cell run while the halo is in flight (spmv_overlapped)
  {
    std::vector<int> ri, rb;
    for (int i = 0; i < ncells; ++i) {
      bool halo = false;
      for (int k = pr.K.ptr[i]; k < pr.K.ptr[i + 1] && !halo; ++k)
        halo = pr.K.col[k] < pr.cell_begin || pr.K.col[k] >= pr.cell_end;
      (halo ? rb : ri).push_back(i);
    }
    n_rows_int = static_cast<int>(ri.size());
    n_rows_bnd = static_cast<int>(rb.size());
    d_rows_int = dmalloc<int>(ri.size());
    d_rows_bnd = dmalloc<int>(rb.size());
    if (!ri.empty()) PDG_CUDA(cudaMemcpy(d_rows_int, ri.data(), ri.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (!rb.empty()) PDG_CUDA(cudaMemcpy(d_rows_bnd, rb.data(), rb.size() * sizeof(int), cudaMemcpyHostToDevice));
    PDG_CUDA(cudaStreamCreateWithFlags(&st_comm, cudaStreamNonBlocking));
    PDG_CUDA(cudaEventCreateWithFlags(&ev_pack, cudaEventDisableTiming));
    PDG_CUDA(cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming));
  }

  // K0 = sum over ranks of the local-row Galerkin products, then the
  // replicated coarse factorisation and the full task list
  if (pr.two_level) {
    double* d_k0 = dmalloc<double>(pr.K0.val.size());
    PDG_CUDA(cudaMemcpyAsync(d_k0, pr.K0.val.data(), pr.K0.val.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    comm_allreduce(d_k0, d_k0, static_cast<long long>(pr.K0.val.size()));
    PDG_CUDA(cudaMemcpyAsync(pr.K0.val.data(), d_k0, pr.K0.val.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_k0);
    finish_coarse(pr);
    upload_tasks();
  }
  PDG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pdg

extern "C" {

int pdg_nccl_unique_id_bytes(void) { return static_cast<int>(sizeof(ncclUniqueId)); }

pdg_status pdg_nccl_get_unique_id(void* id128) {
  return pdg::guarded([&] {
    ncclUniqueId id;
    pdg::nccl_check(pdg::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof id);
  });
}

pdg_status pdg_loopback_create(int world, pdg_loopback** out) {
  return pdg::guarded([&] {
    if (world < 1) throw pdg::ConfigError("loopback: world must be >= 1");
    *out = reinterpret_cast<pdg_loopback*>(new std::shared_ptr<pdg::LoopbackGroup>(
        std::make_shared<pdg::LoopbackGroup>(world)));
  });
}

void pdg_loopback_free(pdg_loopback* g) { delete reinterpret_cast<std::shared_ptr<pdg::LoopbackGroup>*>(g); }

}  // extern "C"
