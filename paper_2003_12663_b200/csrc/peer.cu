// Fused GEMV + all-gather over peer memory for the row-sharded GMRES
// (DESIGN.md 7).  Every rank allocates a replicated vector pair plus a flag
// row with hvb_ipc_alloc, exports a CUDA IPC handle, and opens its peers'
// handles, so each GPU can store straight into every other GPU's vector
// over NVLink.  A matvec is then: k_gemv_f64 with the broadcast epilogue
// (each row result stored into all world replicas), k_peer_signal (system
// fence, then this rank's epoch into every peer's flag row) and
// k_peer_wait (spin until every peer's flag reached the epoch).  The
// vectors alternate by epoch parity; a rank only overwrites parity p after
// every peer signalled the epoch in between, i.e. after they finished
// reading it.  This replaces the GEMV + NCCL all-gather pair of
// parallel.RowGather.
#include <cstdio>

#include "launch.cuh"

namespace hvb {

__global__ void k_peer_signal(unsigned long long* const* flags, int world, int rank, unsigned long long epoch) {
  const int r = threadIdx.x;
  __threadfence_system();
  if (r < world) {
    volatile unsigned long long* f = flags[r] + rank;
    *f = epoch;
  }
  __threadfence_system();
}

// Spins until every peer's epoch arrived; a peer that never signals (a dead
// rank) traps after ~2^35 cycles (~17 s) so the job fails loudly instead of
// hanging the GPU.
__global__ void k_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch) {
  const int r = threadIdx.x;
  if (r < world) {
    const volatile unsigned long long* f = flags + r;
    const long long t0 = clock64();
    while (*f < epoch) {
      if (clock64() - t0 > (1ll << 35)) {
        printf("hvb_peer_wait: rank %d never signalled epoch %llu\n", r, epoch);
        __trap();
      }
    }
  }
  __threadfence_system();
}

cudaError_t launch_peer_signal(unsigned long long* const* flags, int world, int rank, unsigned long long epoch,
                               cudaStream_t st) {
  k_peer_signal<<<1, 32, 0, st>>>(flags, world, rank, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch, cudaStream_t st) {
  k_peer_wait<<<1, 32, 0, st>>>(flags, world, epoch);
  return cudaGetLastError();
}

}  // namespace hvb

