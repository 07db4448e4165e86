// Fused GEMV + all-gather over peer memory for the row-sharded GMRES
// (DESIGN.md 7).  Every rank allocates a replicated vector pair plus a flag
// row with hvb_ipc_alloc, exports a CUDA IPC handle, and opens its peers'
// handles, so each GPU can store straight into every other GPU's vector
// over NVLink.  A matvec is ONE GEMV launch (csrc/gemv.cu, hvb_gemv_bcast):
// every row result is stored into all world replicas, and the last CTA
// publishes the epoch into every rank's flag row with a system-scope
// release store after the CTAs' system fences (peer_release).  k_peer_wait
// then spins with system-scope ACQUIRE loads until every peer's epoch
// arrived, so the rows it guards are visible.  The vectors alternate by
// epoch parity; a rank only overwrites parity p after every peer signalled
// the epoch in between, i.e. after they finished reading it.  This replaces
// the GEMV + NCCL all-gather pair of parallel.RowGather.
#include <cstdio>

#include "launch.cuh"

namespace hvb {

// Spins until every peer's epoch arrived; a peer that never signals (a dead
// rank) traps after ~2^35 cycles (~17 s) so the job fails loudly instead of
// hanging the GPU.
__global__ void k_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch) {
  const int r = threadIdx.x;
  if (r < world) {
    const unsigned long long* f = flags + r;
    const long long t0 = clock64();
    unsigned long long v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= epoch) break;
      if (clock64() - t0 > (1ll << 35)) {
        printf("hvb_peer_wait: rank %d never signalled epoch %llu\n", r, epoch);
        __trap();
      }
    }
  }
  __syncthreads();  // every peer's acquire precedes the kernels that read the vector
}

cudaError_t launch_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch, cudaStream_t st) {
  k_peer_wait<<<1, 32, 0, st>>>(flags, world, epoch);
  return cudaGetLastError();
}

}  // namespace hvb
