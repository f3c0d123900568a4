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

void DeviceSim::comm_allreduce(const double* src, double* dst, long long count) {
  nccl_check(nccl().AllReduce(src, dst, static_cast<size_t>(count), ncclFloat64, ncclSum,
                              static_cast<ncclComm_t>(comm), st),
             "ncclAllReduce");
}

void DeviceSim::comm_exchange(double* v) {
  auto& api = nccl();
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (const HaloPeer& h : halo_peers) {
    if (h.send_count)
      nccl_check(api.Send(d_sendbuf + static_cast<long long>(h.send_off) * b, static_cast<size_t>(h.send_count) * b,
                          ncclFloat64, h.peer, static_cast<ncclComm_t>(comm), st),
                 "ncclSend");
    if (h.recv_count)
      nccl_check(api.Recv(v + (static_cast<long long>(ncells) + h.recv_off) * b, static_cast<size_t>(h.recv_count) * b,
                          ncclFloat64, h.peer, static_cast<ncclComm_t>(comm), st),
                 "ncclRecv");
  }
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

void DeviceSim::comm_destroy() {
  if (comm) {
    nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    comm = nullptr;
  }
}

void DeviceSim::attach_comm(const void* id128, int r, int w) {
  Problem& pr = *P;
  if (w != pr.cfg.world || r != pr.cfg.rank)
    throw ConfigError("attach_comm: rank/world differ from the configuration the problem was built for");
  if (w == 1) return;
  // K0 below is all-reduced in place: a second attach would scale it by world
  if (comm) throw ConfigError("attach_comm: a communicator is already attached");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  PDG_CUDA(cudaSetDevice(pr.cfg.device));
  nccl_check(nccl().CommInitRank(&c, w, id, r), "ncclCommInitRank");
  comm = c;
  d_dot_local = dmalloc<double>(1);
  d_dot_global = dmalloc<double>(1);

  // halo plan from the global mesh adjacency (identical on every rank, host/pack.cpp)
  std::vector<std::vector<int>> send, recv;
  halo_plan(pr, send, recv);
  std::vector<int> send_cells;
  halo_peers.clear();
  for (int peer = 0; peer < w; ++peer) {
    if (peer == r) continue;
    const auto& s = send[peer];
    HaloPeer h{peer, static_cast<int>(send_cells.size()), static_cast<int>(s.size()), 0, 0};
    send_cells.insert(send_cells.end(), s.begin(), s.end());
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

}  // extern "C"
