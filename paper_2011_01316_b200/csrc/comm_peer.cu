// Device-resident communicator of the slab-partitioned path: the two
// collectives the partitioned phi engine needs — the ~2 KB sum / max allreduce of the
// Gram-Schmidt dots and norms after every reducing kernel, and the neighbour halo of one
// element layer before every operator application — as plain kernels over peer memory, so
// they can be recorded into the engine's CUDA graphs (WHILE-node control, no host round-trip
// per Krylov cycle) instead of the host-stepped NCCL path.
//
// Every rank owns one region (PeerLayout): epoch flags written by its peers, its own epoch
// counters, an allreduce inbox [2 parities][ranks][kPeerRed] and halo inboxes
// [2 parities][lo, hi][halo_cap].  A collective of epoch e: each rank stores its payload into
// the peers' inboxes (P2P stores over NVLink for one process per GPU; plain stores when the
// ranks are threads of one process on one device), __threadfence_system, then a release store
// of e into each peer's flag slot; then it waits (acquire) until its own flags reach e and
// reduces the inbox in rank order — every rank gets identical bits.  Two parities suffice: a
// rank can only run ahead into epoch e + 1 after every peer has flagged e, i.e. finished reading
// epoch e - 1.
//
// Regions: one process per GPU exports its region with cudaIpcGetMemHandle and maps the peers'
// (expdg_ctx_peer_export / expdg_ctx_attach_peer); ranks driven by threads of one process share
// a group allocated on the device (expdg_peer_group_create / expdg_ctx_attach_peer_local).
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.cuh"
#include "expdg_internal.cuh"

namespace expdg {

namespace {

constexpr int kPeerMax = 16;
constexpr int kPeerRed = 320;  // doubles per allreduce payload (PhiState::Red is 269)

struct PeerLayout {
  long long halo_cap = 0;
  // offsets in 8-byte words
  static constexpr long long kRedFlag = 0;                   // [kPeerMax]
  static constexpr long long kHaloFlag = kPeerMax;           // [2]
  static constexpr long long kRedEpoch = kPeerMax + 2;
  static constexpr long long kHaloEpoch = kPeerMax + 3;
  static constexpr long long kErr = kPeerMax + 4;            // sticky: a wait for a peer timed out
  static constexpr long long kRedIn = 32;                    // [2][kPeerMax][kPeerRed]
  static constexpr long long kHaloIn = kRedIn + 2LL * kPeerMax * kPeerRed;  // [2][2][halo_cap]
  long long words() const { return kHaloIn + 4 * halo_cap; }
};

struct PeerView {
  unsigned long long* mine;
  unsigned long long* peer[kPeerMax];
  int rank, size;
  long long halo_cap;
  unsigned long long wait_ns;  // bound of every wait for a peer (EXPDG_PEER_TIMEOUT_MS, default 60 s; 0: none)
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded wait for a peer's flag to reach epoch e.  A peer that never arrives (a rank that died,
// or ranks sharing one device whose kernels the hardware does not run at the same time) must
// not hang the GPU: after v.wait_ns the wait gives up, records the epoch in the sticky error
// word (the host turns it into a CommError, PeerComm::check) and every later wait returns at once.
__device__ __forceinline__ void peer_wait(const PeerView& v, const unsigned long long* flag, unsigned long long e) {
  if (ld_acquire_sys(flag) >= e) return;
  if (ld_acquire_sys(v.mine + PeerLayout::kErr) != 0) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(flag) < e) {
    if (global_ns() - t0 > v.wait_ns) {
      st_release_sys(v.mine + PeerLayout::kErr, e);
      return;
    }
  }
}

// count <= kPeerRed elements of 8 (F64) or 4 (I32) bytes; send / recv may alias
__global__ void __launch_bounds__(256) k_peer_allreduce(PeerView v, const void* send, void* recv, int count,
                                                        int type, int op) {
  __shared__ unsigned long long s_e;
  const int tid = threadIdx.x;
  if (tid == 0) s_e = ++v.mine[PeerLayout::kRedEpoch];
  __syncthreads();
  const unsigned long long e = s_e;
  const long long par = (long long)(e & 1);
  for (int i = tid; i < count; i += blockDim.x) {
    unsigned long long w;
    if (type == COMM_F64) w = __double_as_longlong(reinterpret_cast<const double*>(send)[i]);
    else w = (unsigned long long)(unsigned int)reinterpret_cast<const int*>(send)[i];
    for (int r = 0; r < v.size; ++r)
      v.peer[r][PeerLayout::kRedIn + (par * kPeerMax + v.rank) * kPeerRed + i] = w;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (int r = 0; r < v.size; ++r) st_release_sys(v.peer[r] + PeerLayout::kRedFlag + v.rank, e);
  }
  if (tid < v.size) peer_wait(v, v.mine + PeerLayout::kRedFlag + tid, e);
  __syncthreads();
  for (int i = tid; i < count; i += blockDim.x) {
    const unsigned long long* in = v.mine + PeerLayout::kRedIn + par * kPeerMax * kPeerRed + i;
    if (type == COMM_F64) {
      double a = 0.0;
      for (int r = 0; r < v.size; ++r) {  // fixed rank order: identical bits on every rank
        const double x = __longlong_as_double((long long)__ldcv(in + (long long)r * kPeerRed));
        a = r == 0 ? x : (op == COMM_SUM ? a + x : fmax(a, x));
      }
      reinterpret_cast<double*>(recv)[i] = a;
    } else {
      int a = 0;
      for (int r = 0; r < v.size; ++r) {
        const int x = (int)(unsigned int)__ldcv(in + (long long)r * kPeerRed);
        a = r == 0 ? x : (op == COMM_SUM ? a + x : max(a, x));
      }
      reinterpret_cast<int*>(recv)[i] = a;
    }
  }
}

// halo, 1/3: my first / last layer into the lower / upper neighbour's hi / lo inbox of the
// next epoch's parity
__global__ void k_peer_halo_send(PeerView v, const double* send_lo, const double* send_hi, long long count) {
  const long long par = (long long)((v.mine[PeerLayout::kHaloEpoch] + 1) & 1);
  const int lo = (v.rank - 1 + v.size) % v.size, hi = (v.rank + 1) % v.size;
  double* to_lo = reinterpret_cast<double*>(v.peer[lo] + PeerLayout::kHaloIn) + (par * 2 + 1) * v.halo_cap;
  double* to_hi = reinterpret_cast<double*>(v.peer[hi] + PeerLayout::kHaloIn) + (par * 2 + 0) * v.halo_cap;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    to_lo[i] = send_lo[i];
    to_hi[i] = send_hi[i];
  }
}
// halo, 2/3: the epoch's flags to the two neighbours, then wait for theirs
__global__ void k_peer_halo_flag(PeerView v) {
  if (threadIdx.x != 0) return;
  const unsigned long long e = ++v.mine[PeerLayout::kHaloEpoch];
  const int lo = (v.rank - 1 + v.size) % v.size, hi = (v.rank + 1) % v.size;
  __threadfence_system();
  st_release_sys(v.peer[lo] + PeerLayout::kHaloFlag + 1, e);  // lands in its hi inbox
  st_release_sys(v.peer[hi] + PeerLayout::kHaloFlag + 0, e);  // lands in its lo inbox
  peer_wait(v, v.mine + PeerLayout::kHaloFlag + 0, e);
  peer_wait(v, v.mine + PeerLayout::kHaloFlag + 1, e);
}
// halo, 3/3: the inboxes of this epoch into the operator's receive buffers
__global__ void k_peer_halo_recv(PeerView v, double* recv_lo, double* recv_hi, long long count) {
  const long long par = (long long)(v.mine[PeerLayout::kHaloEpoch] & 1);
  const double* in = reinterpret_cast<const double*>(v.mine + PeerLayout::kHaloIn);
  const double* from_lo = in + (par * 2 + 0) * v.halo_cap;
  const double* from_hi = in + (par * 2 + 1) * v.halo_cap;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    recv_lo[i] = __ldcv(from_lo + i);
    recv_hi[i] = __ldcv(from_hi + i);
  }
}

// host barrier of the ranks of one process (see Comm::host_barrier)
struct HostBarrier {
  int size = 1, arrived = 0;
  long long gen = 0;
  std::mutex m;
  std::condition_variable cv;
  void wait() {
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

class PeerComm : public Comm {
 public:
  PeerView v{};
  std::shared_ptr<void> keep;  // the group (threads of one process) or the IPC mappings
  HostBarrier* hb = nullptr;   // threads of one process sharing the device
  PeerComm(const PeerView& view, std::shared_ptr<void> k, HostBarrier* b) : v(view), keep(std::move(k)), hb(b) {
    rank = v.rank;
    size = v.size;
    // 60 s: far above any skew between ranks that entered the same call (the collectives of one
    // Krylov cycle are microseconds apart), short enough that a dead peer ends the run; 0 = unbounded
    long long ms = 60000;
    if (const char* e = std::getenv("EXPDG_PEER_TIMEOUT_MS")) ms = std::max(0LL, std::atoll(e));
    v.wait_ns = ms == 0 ? ~0ull : (unsigned long long)ms * 1000000ull;
  }
  bool graph_capturable() const override { return true; }
  void host_barrier() override {
    if (hb) hb->wait();
  }
  void allreduce(const void* send, void* recv, long long count, int type, int op, cudaStream_t s) override {
    if (count > kPeerRed) throw CommError("peer allreduce: payload above " + std::to_string(kPeerRed) + " words");
    k_peer_allreduce<<<1, 256, 0, s>>>(v, send, recv, (int)count, type, op);
    EXPDG_CUDA(cudaGetLastError());
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, long long count,
            cudaStream_t s) override {
    if (count > v.halo_cap)
      throw CommError("peer halo: layer of " + std::to_string(count) + " doubles above the group's capacity " +
                      std::to_string(v.halo_cap));
    const int g = (int)std::max<long long>(1, std::min<long long>(592, (count + 255) / 256));
    k_peer_halo_send<<<g, 256, 0, s>>>(v, send_lo, send_hi, count);
    k_peer_halo_flag<<<1, 32, 0, s>>>(v);
    k_peer_halo_recv<<<g, 256, 0, s>>>(v, recv_lo, recv_hi, count);
    EXPDG_CUDA(cudaGetLastError());
  }
  const char* kind() const override { return "peer"; }
  void check() override {
    unsigned long long err = 0;
    EXPDG_CUDA(cudaMemcpy(&err, v.mine + PeerLayout::kErr, sizeof(err), cudaMemcpyDeviceToHost));
    if (err == 0) return;
    EXPDG_CUDA(cudaMemset(v.mine + PeerLayout::kErr, 0, sizeof(err)));
    throw CommError("peer communicator: rank " + std::to_string(rank) + " waited " +
                    std::to_string(v.wait_ns / 1000000ull) + " ms for a peer at epoch " +
                    std::to_string(err) + " (a rank that stopped, or ranks sharing one device that did not run "
                    "concurrently); the results of this call are invalid");
  }
};

}  // namespace

// ---- ranks = threads of one process, one device
struct PeerGroup {
  int size = 1;
  PeerLayout lay;
  std::vector<unsigned long long*> region;
  HostBarrier barrier;
  ~PeerGroup() {
    for (auto* r : region) cudaFree(r);
  }
};

std::shared_ptr<PeerGroup> make_peer_group(int size, long long halo_cap) {
  if (size < 1 || size > kPeerMax) throw std::invalid_argument("peer group: 1 <= size <= 16");
  if (halo_cap < 0) throw std::invalid_argument("peer group: negative halo capacity");
  auto g = std::make_shared<PeerGroup>();
  g->size = size;
  g->barrier.size = size;
  g->lay.halo_cap = halo_cap;
  g->region.resize(size, nullptr);
  for (int r = 0; r < size; ++r) {
    EXPDG_CUDA(cudaMalloc(&g->region[r], sizeof(unsigned long long) * g->lay.words()));
    EXPDG_CUDA(cudaMemset(g->region[r], 0, sizeof(unsigned long long) * g->lay.words()));
  }
  return g;
}

std::unique_ptr<Comm> make_peer_comm_local(const std::shared_ptr<PeerGroup>& g, int rank) {
  if (!g || rank < 0 || rank >= g->size) throw std::invalid_argument("peer comm: bad rank");
  PeerView v{};
  v.mine = g->region[rank];
  for (int r = 0; r < g->size; ++r) v.peer[r] = g->region[r];
  v.rank = rank;
  v.size = g->size;
  v.halo_cap = g->lay.halo_cap;
  return std::make_unique<PeerComm>(v, g, &g->barrier);
}

// ---- one process per GPU: this rank's region, exported with a CUDA IPC handle
struct PeerExport {
  int size = 1;
  PeerLayout lay;
  unsigned long long* region = nullptr;
  std::vector<void*> opened;
  ~PeerExport() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    cudaFree(region);
  }
};

std::shared_ptr<PeerExport> make_peer_export(int size, long long halo_cap, unsigned char handle_out[64]) {
  if (size < 1 || size > kPeerMax) throw std::invalid_argument("peer export: 1 <= size <= 16");
  auto x = std::make_shared<PeerExport>();
  x->size = size;
  x->lay.halo_cap = halo_cap;
  EXPDG_CUDA(cudaMalloc(&x->region, sizeof(unsigned long long) * x->lay.words()));
  EXPDG_CUDA(cudaMemset(x->region, 0, sizeof(unsigned long long) * x->lay.words()));
  cudaIpcMemHandle_t h;
  EXPDG_CUDA(cudaIpcGetMemHandle(&h, x->region));
  static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
  std::memcpy(handle_out, &h, 64);
  return x;
}

std::unique_ptr<Comm> make_peer_comm_ipc(const std::shared_ptr<PeerExport>& x, const unsigned char* handles,
                                         int rank, int size) {
  if (!x || size != x->size || rank < 0 || rank >= size) throw std::invalid_argument("peer comm: bad rank / size");
  PeerView v{};
  v.mine = x->region;
  for (int r = 0; r < size; ++r) {
    if (r == rank) {
      v.peer[r] = x->region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * (size_t)r, 64);
    void* p = nullptr;
    EXPDG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    x->opened.push_back(p);
    v.peer[r] = static_cast<unsigned long long*>(p);
  }
  v.rank = rank;
  v.size = size;
  v.halo_cap = x->lay.halo_cap;
  return std::make_unique<PeerComm>(v, x, nullptr);
}

}  // namespace expdg
