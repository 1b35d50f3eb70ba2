// Step barrier + max-reduction over NVLink peer memory (the fused ghost
// refresh's ordering point, exports.py).  After a rank's step kernel it
// publishes its guard displacement and the step's epoch number into every
// peer's mailbox (CUDA-IPC mapped), then waits until every peer has published
// the same epoch, and replaces its value with the maximum.  Kernel completion
// of the step kernel precedes the publication in stream order, so a peer that
// passes the barrier sees all ghost copies this rank wrote into its buffers,
// and this rank cannot overwrite a buffer a peer is still reading.
//
// Mailbox (int64): [parity][src][{epoch, value bits}] with parity = epoch & 1,
// so a publication for epoch e + 1 never lands on the slot a slow peer is
// still reading for epoch e.  A peer that does not arrive within the caller's
// timeout (globaltimer nanoseconds; the host sets it, default 120 s, so a rank
// whose host pauses between steps -- a trajectory dump, a GC pass -- does not
// abort its peers) is a protocol error (status word), never a hang.
#include "tmd_common.cuh"

namespace tmd {

constexpr int kMailPeers = 8;

struct Mailboxes {
  long long* box[kMailPeers];
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_peer_sync(long long epoch, int me, int n, Mailboxes M, double* __restrict__ value,
                            unsigned long long timeout_ns, int64_t* __restrict__ st) {
  __shared__ double vals[kMailPeers];
  const int q = threadIdx.x;
  const int par = (int)(epoch & 1);
  const double mine = *value;
  if (q < n) {
    volatile long long* slot = M.box[q] + ((par * kMailPeers + me) * 2);
    slot[1] = __double_as_longlong(mine);
    __threadfence_system();
    slot[0] = epoch;
  }
  __syncthreads();
  if (q < n) {
    volatile long long* in = M.box[me] + ((par * kMailPeers + q) * 2);
    const unsigned long long t0 = global_ns();
    bool ok = true;
    while (in[0] < epoch) {
      if (global_ns() - t0 > timeout_ns) {
        ok = false;
        break;
      }
    }
    __threadfence_system();
    vals[q] = ok ? __longlong_as_double(in[1]) : 0.0;
    if (!ok) raise_status(st, TMD_PROTOCOL, (unsigned long long)q);
  }
  __syncthreads();
  if (q == 0) {
    double m = mine;
    for (int r = 0; r < n; ++r) m = fmax(m, vals[r]);
    *value = m;
  }
}

// Small all-gather over the same mailboxes (the epoch's count exchanges at
// P > 1): every rank publishes w <= kGatherWords int64 values into every
// peer's gather slot [parity][me] (values, fence, then the call's stamp) and
// collects the n slots of its own mailbox into out (n, w).  Parity by call
// number, as the barrier: a rank publishes call e + 2 only after every peer
// published e + 1, which each does after it finished reading call e.
constexpr int kBarrierWords = 2 * kMailPeers * 2;
constexpr int kGatherWords = 24;
constexpr int kGatherSlot = 1 + kGatherWords;

__global__ void k_peer_allgather(long long epoch, int me, int n, Mailboxes M, const long long* __restrict__ in, int w,
                                 long long* __restrict__ out, unsigned long long timeout_ns, int64_t* __restrict__ st) {
  const int q = threadIdx.x;
  const int par = (int)(epoch & 1);
  if (q < n) {
    volatile long long* slot = M.box[q] + kBarrierWords + (par * kMailPeers + me) * kGatherSlot;
    for (int k = 0; k < w; ++k) slot[1 + k] = in[k];
    __threadfence_system();
    slot[0] = epoch;
  }
  __syncthreads();
  if (q < n) {
    volatile long long* src = M.box[me] + kBarrierWords + (par * kMailPeers + q) * kGatherSlot;
    const unsigned long long t0 = global_ns();
    bool ok = true;
    while (src[0] < epoch) {
      if (global_ns() - t0 > timeout_ns) {
        ok = false;
        break;
      }
    }
    __threadfence_system();
    for (int k = 0; k < w; ++k) out[q * w + k] = ok ? src[1 + k] : 0;
    if (!ok) raise_status(st, TMD_PROTOCOL, (unsigned long long)q);
  }
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_peer_allgather(int64_t epoch, int32_t me, int32_t n_peers, int64_t* const* h_mailbox,
                                  const int64_t* d_in, int32_t w, int64_t* d_out, double timeout_s, int64_t* d_status,
                                  void* stream) {
  if (n_peers < 1 || n_peers > kMailPeers || me < 0 || me >= n_peers || !h_mailbox || epoch < 1 || w < 0 ||
      w > kGatherWords || (w > 0 && (!d_in || !d_out)) || !(timeout_s > 0.0))
    return TMD_ERR_ARG;
  Mailboxes M{};
  for (int r = 0; r < n_peers; ++r) {
    if (!h_mailbox[r]) return TMD_ERR_ARG;
    M.box[r] = reinterpret_cast<long long*>(h_mailbox[r]);
  }
  const unsigned long long ns = timeout_s >= 1.8e10 ? ~0ULL : (unsigned long long)(timeout_s * 1e9);
  k_peer_allgather<<<1, 32, 0, as_stream(stream)>>>((long long)epoch, me, n_peers, M,
                                                    reinterpret_cast<const long long*>(d_in), w,
                                                    reinterpret_cast<long long*>(d_out), ns, d_status);
  TMD_LAUNCH_CHECK("peer_allgather");
  return TMD_OK;
}

extern "C" int tmd_peer_gather_words(void) { return kGatherWords; }

extern "C" int tmd_peer_sync(int64_t epoch, int32_t me, int32_t n_peers, int64_t* const* h_mailbox, double* d_value,
                             double timeout_s, int64_t* d_status, void* stream) {
  if (n_peers < 1 || n_peers > kMailPeers || me < 0 || me >= n_peers || !h_mailbox || !d_value || epoch < 1 ||
      !(timeout_s > 0.0))
    return TMD_ERR_ARG;
  Mailboxes M{};
  for (int r = 0; r < n_peers; ++r) {
    if (!h_mailbox[r]) return TMD_ERR_ARG;
    M.box[r] = reinterpret_cast<long long*>(h_mailbox[r]);
  }
  const unsigned long long ns = timeout_s >= 1.8e10 ? ~0ULL : (unsigned long long)(timeout_s * 1e9);
  k_peer_sync<<<1, 32, 0, as_stream(stream)>>>((long long)epoch, me, n_peers, M, d_value, ns, d_status);
  TMD_LAUNCH_CHECK("peer_sync");
  return TMD_OK;
}

extern "C" int tmd_mailbox_words(void) { return kBarrierWords + 2 * kMailPeers * kGatherSlot; }
