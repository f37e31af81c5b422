// Cluster / async-copy primitives (inline PTX, sm_90+ semantics, used on sm_100a):
// DSMEM remote stores, mbarriers signalled across the cluster, split cluster barriers and
// cp.async for staging small read-only tables into SMEM.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace cssar {

CSSAR_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async 16-byte chunks (L2 only, no L1 allocation); completion via cp_async_wait_all()
CSSAR_DEV void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
CSSAR_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// copy n (even) float2 from global to SMEM asynchronously
CSSAR_DEV void copy_table_async(float2* dst, const float2* src, int n, int t, int nthreads) {
  for (int i = t; i < n / 2; i += nthreads) cp_async16(dst + 2 * i, src + 2 * i);
}

CSSAR_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CSSAR_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

CSSAR_DEV void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
CSSAR_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }

// address of the same SMEM offset in CTA `rank` of this cluster (shared::cluster window)
CSSAR_DEV uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}

CSSAR_DEV void st_cluster(uint32_t raddr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};\n" ::"r"(raddr), "f"(v.x), "f"(v.y) : "memory");
}

// arrive (release, cluster scope) on an mbarrier that lives in another CTA of the cluster
CSSAR_DEV void mbar_arrive_remote(uint32_t raddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(raddr) : "memory");
}

// wait (acquire, cluster scope) until the phase with the given parity has completed
CSSAR_DEV void mbar_wait(const uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// Programmatic dependent launch (sm_90+): kernels of the ITA loop are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so the next kernel's CTAs can start (SMEM
// tables, mbarrier set-up) while this one drains; pdl_wait() blocks until the previous kernel
// has completed and its memory is visible (a no-op without the attribute).
CSSAR_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
CSSAR_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

CSSAR_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

}  // namespace cssar
