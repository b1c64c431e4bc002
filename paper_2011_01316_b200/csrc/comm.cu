// NCCL and host-staged communicators (see comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.cuh"
#include "expdg_internal.cuh"

namespace expdg {

// ---------------------------------------------------------------- NCCL (loaded lazily)
// NCCL is resolved at run time with dlopen so this library carries no link-time
// dependency on a particular libnccl: inside a PyTorch process the copy torch
// already loaded is reused.
namespace {
struct NcclApi {
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

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  });
  if (!api.CommInitRank || !api.AllReduce || !api.Send || !api.Recv)
    throw CommError("NCCL: libnccl.so.2 not found (needed for the multi-GPU slab path)");
  return api;
}

void ncheck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CommError(std::string("NCCL ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

class NcclComm : public Comm {
 public:
  ncclComm_t c = nullptr;
  NcclComm(const void* uid, int r, int n) {
    rank = r;
    size = n;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncheck(nccl().CommInitRank(&c, n, id, r), "CommInitRank");
  }
  ~NcclComm() override {
    if (c) nccl().CommDestroy(c);
  }
  void allreduce(const void* send, void* recv, long long count, int type, int op, cudaStream_t s) override {
    ncheck(nccl().AllReduce(send, recv, (size_t)count, type == COMM_F64 ? ncclFloat64 : ncclInt32,
                            op == COMM_SUM ? ncclSum : ncclMax, c, s),
           "AllReduce");
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, long long count,
            cudaStream_t s) override {
    if (size == 1) {  // periodic wrap onto itself
      EXPDG_CUDA(cudaMemcpyAsync(recv_hi, send_lo, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
      EXPDG_CUDA(cudaMemcpyAsync(recv_lo, send_hi, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
      return;
    }
    const int lo = (rank - 1 + size) % size, hi = (rank + 1) % size;
    const NcclApi& a = nccl();
    ncheck(a.GroupStart(), "GroupStart");
    ncheck(a.Send(send_lo, (size_t)count, ncclFloat64, lo, c, s), "Send");
    ncheck(a.Recv(recv_hi, (size_t)count, ncclFloat64, hi, c, s), "Recv");
    ncheck(a.Send(send_hi, (size_t)count, ncclFloat64, hi, c, s), "Send");
    ncheck(a.Recv(recv_lo, (size_t)count, ncclFloat64, lo, c, s), "Recv");
    ncheck(a.GroupEnd(), "GroupEnd");
  }
  const char* kind() const override { return "nccl"; }
};
}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int size) {
  if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("nccl comm: bad rank / size");
  return std::make_unique<NcclComm>(unique_id, rank, size);
}

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  ncheck(nccl().GetUniqueId(&id), "GetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

// ---------------------------------------------------------------- host-staged group
struct LocalGroup {
  int size = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<std::vector<char>> stage;
  std::vector<std::vector<double>> lo, hi;
  explicit LocalGroup(int n) : size(n), stage(n), lo(n), hi(n) {}
  void barrier() {
    std::unique_lock<std::mutex> l(m);
    const long long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return gen != g; });
    }
  }
};

std::shared_ptr<LocalGroup> make_local_group(int size) {
  if (size < 1) throw std::invalid_argument("local group: size must be positive");
  return std::make_shared<LocalGroup>(size);
}

namespace {
class LocalComm : public Comm {
 public:
  std::shared_ptr<LocalGroup> g;
  LocalComm(const std::shared_ptr<LocalGroup>& grp, int r) : g(grp) {
    rank = r;
    size = grp->size;
  }
  void allreduce(const void* send, void* recv, long long count, int type, int op, cudaStream_t s) override {
    const size_t esz = type == COMM_F64 ? 8 : 4;
    std::vector<char>& mine = g->stage[rank];
    mine.resize(esz * count);
    EXPDG_CUDA(cudaMemcpyAsync(mine.data(), send, esz * count, cudaMemcpyDeviceToHost, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
    g->barrier();
    std::vector<char> out(esz * count);
    for (long long i = 0; i < count; ++i) {  // fixed rank order: identical on every rank
      if (type == COMM_F64) {
        double a = 0.0;
        for (int r = 0; r < size; ++r) {
          const double v = reinterpret_cast<const double*>(g->stage[r].data())[i];
          a = (r == 0) ? v : (op == COMM_SUM ? a + v : (v > a ? v : a));
        }
        reinterpret_cast<double*>(out.data())[i] = a;
      } else {
        int a = 0;
        for (int r = 0; r < size; ++r) {
          const int v = reinterpret_cast<const int*>(g->stage[r].data())[i];
          a = (r == 0) ? v : (op == COMM_SUM ? a + v : (v > a ? v : a));
        }
        reinterpret_cast<int*>(out.data())[i] = a;
      }
    }
    g->barrier();
    EXPDG_CUDA(cudaMemcpyAsync(recv, out.data(), esz * count, cudaMemcpyHostToDevice, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, long long count,
            cudaStream_t s) override {
    g->lo[rank].resize(count);
    g->hi[rank].resize(count);
    EXPDG_CUDA(cudaMemcpyAsync(g->lo[rank].data(), send_lo, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    EXPDG_CUDA(cudaMemcpyAsync(g->hi[rank].data(), send_hi, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
    g->barrier();
    const int up = (rank + 1) % size, dn = (rank - 1 + size) % size;
    EXPDG_CUDA(cudaMemcpyAsync(recv_hi, g->lo[up].data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
    EXPDG_CUDA(cudaMemcpyAsync(recv_lo, g->hi[dn].data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
    g->barrier();
  }
  const char* kind() const override { return "local"; }
};
}  // namespace

std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank) {
  if (!g || rank < 0 || rank >= g->size) throw std::invalid_argument("local comm: bad rank");
  return std::make_unique<LocalComm>(g, rank);
}

}  // namespace expdg
