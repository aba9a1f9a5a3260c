// NCCL implementation of qswg::Comm (one process per GPU, NVLink/NVSwitch).
//
// libnccl.so.2 is resolved with dlopen at communicator creation, so a
// single-GPU process never needs NCCL and a process that already loaded
// torch's bundled NCCL shares that copy (same soname).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/qswg.h"
#include "comm.hpp"
#include "device.hpp"

namespace qswg {

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api = load();
    if (!api.lib) throw CudaError("libnccl.so.2 could not be loaded (needed for multi-GPU runs)");
    return api;
  }

 private:
  static NcclApi load() {
    NcclApi a;
    a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.lib) return a;
    auto sym = [&](const char* n) {
      void* p = dlsym(a.lib, n);
      if (!p) throw CudaError(std::string("NCCL symbol missing: ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw CudaError(std::string("NCCL ") + what + ": " + NcclApi::get().GetErrorString(r));
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(const ncclUniqueId& id, int rank, int world, int device) : rank_(rank), world_(world), device_(device) {
    DeviceGuard g(device);
    nccl_check(NcclApi::get().CommInitRank(&comm_, world, id, rank), "CommInitRank");
  }
  ~NcclComm() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }

  void allgather_rows(void* full, const std::vector<std::int64_t>& starts, std::size_t elem_bytes,
                      cudaStream_t s) override {
    auto& api = NcclApi::get();
    auto* base = static_cast<unsigned char*>(full);
    nccl_check(api.GroupStart(), "GroupStart");
    for (int r = 0; r < world_; ++r) {
      const std::size_t off = static_cast<std::size_t>(starts[static_cast<std::size_t>(r)]) * elem_bytes;
      const std::size_t cnt = static_cast<std::size_t>(starts[static_cast<std::size_t>(r) + 1] -
                                                       starts[static_cast<std::size_t>(r)]) * elem_bytes;
      if (cnt) nccl_check(api.Broadcast(base + off, base + off, cnt, ncclUint8, r, comm_, s), "Broadcast");
    }
    nccl_check(api.GroupEnd(), "GroupEnd");
  }

  void exchange_ranges(void* full, const std::vector<std::vector<std::int64_t>>& lo,
                       const std::vector<std::vector<std::int64_t>>& hi, std::size_t elem_bytes,
                       cudaStream_t s) override {
    auto& api = NcclApi::get();
    auto* base = static_cast<unsigned char*>(full);
    nccl_check(api.GroupStart(), "GroupStart");
    for (int q = 0; q < world_; ++q) {
      if (q == rank_) continue;
      const auto uq = static_cast<std::size_t>(q), ur = static_cast<std::size_t>(rank_);
      // what peer q needs from me
      if (hi[uq][ur] > lo[uq][ur]) {
        nccl_check(api.Send(base + lo[uq][ur] * elem_bytes, static_cast<std::size_t>(hi[uq][ur] - lo[uq][ur]) * elem_bytes,
                            ncclUint8, q, comm_, s), "Send");
      }
      // what I need from peer q
      if (hi[ur][uq] > lo[ur][uq]) {
        nccl_check(api.Recv(base + lo[ur][uq] * elem_bytes, static_cast<std::size_t>(hi[ur][uq] - lo[ur][uq]) * elem_bytes,
                            ncclUint8, q, comm_, s), "Recv");
      }
    }
    nccl_check(api.GroupEnd(), "GroupEnd");
  }

  void allreduce_max_u64(unsigned long long* buf, std::size_t n, cudaStream_t s) override {
    nccl_check(NcclApi::get().AllReduce(buf, buf, n, ncclUint64, ncclMax, comm_, s), "AllReduce");
  }

  void allreduce_sum_f64(double* buf, std::size_t n, cudaStream_t s) override {
    nccl_check(NcclApi::get().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, s), "AllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_, world_, device_;
};

}  // namespace

}  // namespace qswg

namespace qswg {

Comm* comm_from_handle(qswg_comm* c) { return c ? c->c.get() : nullptr; }

int comm_unique_id_size() { return NCCL_UNIQUE_ID_BYTES; }

int comm_get_unique_id(uint8_t* id) {
  ncclUniqueId uid;
  nccl_check(NcclApi::get().GetUniqueId(&uid), "GetUniqueId");
  std::memcpy(id, uid.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int comm_create(const uint8_t* id, int rank, int world, int device, qswg_comm** out) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("invalid rank/world");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  auto h = std::make_unique<qswg_comm>();
  h->c = std::make_unique<NcclComm>(uid, rank, world, device);
  *out = h.release();
  return 0;
}

void comm_destroy(qswg_comm* c) { delete c; }

}  // namespace qswg
