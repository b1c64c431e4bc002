// Communicators of the slab-partitioned device path.
//
// The partitioned phi engine needs exactly two collectives:
//   * a sum-allreduce of the reduced Gram-Schmidt dots / norms after every
//     reducing kernel (max-allreduce for the per-step max|u| and flags), and
//   * a periodic neighbour exchange of one element row (face-trace halo) before
//     every operator application.
// NcclComm runs them on the stream through NCCL over NVLink / NVSwitch (one
// process per GPU).  LocalComm is a host-staged implementation for several
// ranks driven by threads of ONE process (tests on a single GPU: the ranks'
// kernels never wait on each other on the device, the host threads meet at
// barriers).
#pragma once

#include <cuda_runtime.h>

#include <memory>

namespace expdg {

enum CommType { COMM_F64 = 0, COMM_I32 = 1 };
enum CommOp { COMM_SUM = 0, COMM_MAX = 1 };

class Comm {
 public:
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // recv = op over ranks of send (device buffers, may alias), ordered on s
  virtual void allreduce(const void* send, void* recv, long long count, int type, int op, cudaStream_t s) = 0;
  // periodic neighbour exchange along the partition axis, ordered on s:
  // send_lo -> rank-1 (lands in its recv_hi), send_hi -> rank+1 (lands in its recv_lo)
  virtual void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, long long count,
                    cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
  // the collectives are plain kernels on the stream (recordable into the engine's CUDA graphs)
  virtual bool graph_capturable() const { return false; }
  // Ranks that share ONE device (threads of one process): a host barrier the library passes
  // before launching device-side collectives, so no rank can sit in a device-synchronising
  // runtime call (cudaFree, pinned allocation) while another rank's collective kernel spins on
  // it.  No-op for one process per GPU.
  virtual void host_barrier() {}
  // After the stream has been synchronised: throws CommError if a device-side collective gave
  // up waiting for a peer (bounded waits, comm_peer.cu).  No-op for the other communicators.
  virtual void check() {}
};

struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int size);
std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank);
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int size);
// device-resident peer-memory communicator (comm_peer.cu)
struct PeerGroup;
struct PeerExport;
std::shared_ptr<PeerGroup> make_peer_group(int size, long long halo_cap);
std::unique_ptr<Comm> make_peer_comm_local(const std::shared_ptr<PeerGroup>& g, int rank);
std::shared_ptr<PeerExport> make_peer_export(int size, long long halo_cap, unsigned char handle_out[64]);
std::unique_ptr<Comm> make_peer_comm_ipc(const std::shared_ptr<PeerExport>& x, const unsigned char* handles,
                                         int rank, int size);
void nccl_unique_id(void* out128);

}  // namespace expdg
