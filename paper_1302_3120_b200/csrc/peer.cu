// Multi-GPU peer-memory plumbing:
//   * flag barrier: every rank release-stores its epoch into a slot of every peer's
//     IPC-mapped workspace and acquire-polls its own slots (system scope) -- replaces the
//     one-word NCCL all-reduce that ordered the fused (peer-store) transposes.  Polls are
//     bounded by a wall-clock timeout that raises an error flag instead of hanging.
//   * the same barrier over all ranks of a single-device emulation group, one block per
//     rank in ONE cooperative launch (the blocks are co-resident, so the spin is legal on one
//     GPU -- unlike separate launches or processes that wait on each other).
//   * CUDA-IPC export / open of a device pointer inside a caching-allocator block (base +
//     offset), and a peer-store test kernel, used by map_peers and by the 2-process test.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>
#include "kernels.cuh"

namespace cssar {

namespace {
constexpr unsigned long long kBarrierTimeoutNs = 20ull * 1000ull * 1000ull * 1000ull;   // 20 s

CSSAR_DEV unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
CSSAR_DEV void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CSSAR_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
}  // namespace

// One barrier round for `rank` (called by one thread): epoch <- epoch + 1, publish it in slot
// [rank] of every rank's slot array, wait until every own slot [q] has reached it.
CSSAR_DEV void flag_barrier_rank(int rank, int world, const PeerSlots& ps, uint32_t* epoch, uint32_t* err) {
  const uint32_t e = *epoch + 1u;
  *epoch = e;
  __threadfence_system();                                   // this rank's earlier writes first
  for (int q = 0; q < world; ++q) st_release_sys(ps.slots[q] + rank, e);
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < world; ++q) {
    const uint32_t* mine = ps.slots[rank] + q;
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      if (global_ns() - t0 > kBarrierTimeoutNs) {
        atomicOr(err, 1u);
        return;
      }
    }
  }
}

__global__ void flag_barrier_kernel(int rank, int world, const PeerSlots ps, uint32_t* epoch, uint32_t* err) {
  if (threadIdx.x == 0 && blockIdx.x == 0) flag_barrier_rank(rank, world, ps, epoch, err);
}

// emulation group: block r is rank r (all blocks co-resident: cooperative launch)
__global__ void flag_barrier_group_kernel(int world, const PeerSlots ps, const EpochPtrs ep, int rounds,
                                          uint32_t* err) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < rounds; ++i) flag_barrier_rank((int)blockIdx.x, world, ps, ep.p[blockIdx.x], err);
}

cudaError_t launch_flag_barrier(int rank, int world, const PeerSlots& ps, uint32_t* epoch, uint32_t* err,
                                cudaStream_t s) {
  flag_barrier_kernel<<<1, 32, 0, s>>>(rank, world, ps, epoch, err);
  return cudaGetLastError();
}

cudaError_t launch_flag_barrier_group(int world, const PeerSlots& ps, const EpochPtrs& ep, int rounds, uint32_t* err,
                                      cudaStream_t s) {
  void* args[] = {(void*)&world, (void*)&ps, (void*)&ep, (void*)&rounds, (void*)&err};
  return cudaLaunchCooperativeKernel((const void*)flag_barrier_group_kernel, dim3((unsigned)world), dim3(32), args,
                                     0, s);
}

// ---- CUDA IPC of a pointer inside an allocation (torch's caching allocator hands out
// offsets into larger cudaMalloc blocks; IPC handles name the block base)
int ipc_export(const void* p, IpcRec* rec) {
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&range), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      range = nullptr;
  }
  *rec = IpcRec{};
  rec->off = ~0ull;
  if (!range || !p) return -1;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return -1;
  if (cudaIpcGetMemHandle(&rec->h, (void*)base) != cudaSuccess) return -1;
  rec->off = (unsigned long long)((CUdeviceptr)p - base);
  return 0;
}

int ipc_open(const IpcRec& rec, void** base_out, void** ptr_out) {
  *base_out = *ptr_out = nullptr;
  if (rec.off == ~0ull) return -1;
  void* b = nullptr;
  if (cudaIpcOpenMemHandle(&b, rec.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return -1;
  *base_out = b;
  *ptr_out = static_cast<char*>(b) + rec.off;
  return 0;
}

__global__ void peer_store_kernel(uint32_t* dst, uint32_t pattern, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = pattern ^ (uint32_t)i;
  __threadfence_system();
}

cudaError_t launch_peer_store(uint32_t* dst, uint32_t pattern, long long n, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  if (blocks < 1) blocks = 1;
  peer_store_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, pattern, n);
  return cudaGetLastError();
}

}  // namespace cssar
