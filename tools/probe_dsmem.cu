// probe_dsmem.cu — cluster DSMEM primitives used by conv_pair.cu, in isolation:
// each CTA of a 2-CTA cluster stores into and arrives on its partner's shared
// memory, then waits on its own barrier.  Variant selects the arrive form.
#include <cstdio>
#include "../paper_2006_10004_b200/csrc/sm100.cuh"
using namespace tvs;

__global__ void k_probe(int variant, int* out) {
  __shared__ uint64_t bar;
  __shared__ __align__(16) uint32_t buf[4];
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    buf[0] = buf[1] = buf[2] = buf[3] = 0;
  }
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x == 0) {
    const uint32_t peer = rank ^ 1;
    const uint32_t rbuf = mapa_shared(smem_u32(buf), peer);
    const uint32_t rbar = mapa_shared(smem_u32(&bar), peer);
    st_cluster_v4(rbuf, 100 + rank, 2, 3, 4);
    if (variant == 2) asm volatile("fence.proxy.async;" ::: "memory");
    if (variant == 3) asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
    if (variant == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (variant != 1) {
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
    }
    uint32_t ok = 0;
    for (int i = 0; i < (1 << 24) && !ok; ++i) {
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
          "selp.b32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
    }
    out[blockIdx.x * 2] = ok;
    out[blockIdx.x * 2 + 1] = buf[0];
  }
  __syncthreads();
  cluster_sync_all();
}

int main() {
  int* d;
  cudaMalloc(&d, 64 * sizeof(int));
  for (int v = 0; v < 5; ++v) {
    cudaMemset(d, 0, 64 * sizeof(int));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4);
    cfg.blockDim = dim3(64);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_probe, v, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d launch %s sync %s  ok/val: %d %d | %d %d | %d %d | %d %d\n", v, cudaGetErrorString(e),
           cudaGetErrorString(e2), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    if (e2 != cudaSuccess) { printf("variant %d failed\n", v); return 1; }
  }
  return 0;
}
