// Probe: where do the rows / columns of a tcgen05.mma accumulator land in TMEM for the
// shapes the grouped GEMM does not use yet (cta_group::1 M=64, cta_group::2 M=128)?
// D[r][c] = (r + 1) + 256 (c + 1) by construction (A[r][0] = r + 1, A[r][1] = 256,
// B[c][0] = 1, B[c][1] = c + 1, other k zero), read back from all 128 lanes x N columns.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2508_12851_b200/csrc \
//        tools/umma_layout_probe.cu -o tools/umma_layout_probe && ./tools/umma_layout_probe
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace mp;

constexpr int N = 64;  // accumulator columns

// K-major SWIZZLE_128B tile of `rows` x 64 bf16 (one 128-byte row each)
__device__ void fill_tile(uint8_t* tile, int rows, bool is_a, int row_base) {
  for (int i = threadIdx.x; i < rows * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    float v = 0.f;
    if (is_a) v = k == 0 ? float(row_base + r + 1) : (k == 1 ? 256.f : 0.f);
    else v = k == 0 ? 1.f : (k == 1 ? float(row_base + r + 1) : 0.f);
    const int chunk = (k * 2) / 16, within = (k * 2) % 16;
    const int off = r * 128 + ((chunk ^ (r & 7)) << 4) + within;
    *reinterpret_cast<__nv_bfloat16*>(tile + off) = __float2bfloat16(v);
  }
}

template <int kPair, int M>
__global__ void __launch_bounds__(128) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;                // A rows of this CTA
  uint8_t* B = sm + 128 * 128;    // B rows of this CTA
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  const uint32_t rank = kPair ? cluster_ctarank() : 0;
  const int a_rows = kPair ? M / 2 : M, b_rows = kPair ? N / 2 : N;
  fill_tile(A, 128, true, int(rank) * a_rows);
  fill_tile(B, 64, false, int(rank) * b_rows);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    if (kPair) tmem_alloc_2sm<256>(&tslot);
    else tmem_alloc<256>(&tslot);
  }
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = make_idesc_bf16(M, N);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = make_sdesc_sw128(smem_u32(A)) + uint64_t(2 * ks);
      const uint64_t bd = make_sdesc_sw128(smem_u32(B)) + uint64_t(2 * ks);
      if (kPair) umma_bf16_2sm(tmem, ad, bd, idesc, ks ? 1u : 0u);
      else umma_bf16(tmem, ad, bd, idesc, ks ? 1u : 0u);
    }
    if (kPair) umma_commit_2sm_mc(&done, 0x3);
    else umma_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j)
      out[(size_t(rank) * 128 + warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (kPair) tmem_dealloc_2sm<256>(tmem);
    else tmem_dealloc<256>(tmem);
  }
}

template <int kPair, int M>
void run(const char* name) {
  float* d;
  const int ctas = kPair ? 2 : 1;
  cudaMalloc(&d, size_t(ctas) * 128 * N * 4);
  cudaMemset(d, 0, size_t(ctas) * 128 * N * 4);
  cudaFuncSetAttribute(probe<kPair, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, probe<kPair, M>, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  printf("== %s: %s\n", name, cudaGetErrorString(e));
  std::vector<float> h(size_t(ctas) * 128 * N);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  for (int cta = 0; cta < ctas; ++cta)
    for (int lane = 0; lane < 128; ++lane) {
      // summarise one lane: the (row, col) pairs in its first columns
      std::vector<int> rows, cols;
      for (int c = 0; c < N; ++c) {
        const int v = int(h[(size_t(cta) * 128 + lane) * N + c]);
        if (v == 0) { rows.push_back(-1); cols.push_back(-1); continue; }
        rows.push_back(v % 256 - 1);
        cols.push_back(v / 256 - 1);
      }
      printf("cta %d lane %3d: ", cta, lane);
      for (int c = 0; c < N; c += 8) printf("[c%2d r%3d col%3d] ", c, rows[c], cols[c]);
      printf("\n");
    }
  cudaFree(d);
}

int main() {
  run<0, 128>("cta_group::1 M=128 (reference)");
  run<0, 64>("cta_group::1 M=64");
  run<1, 256>("cta_group::2 M=256 (reference)");
  run<1, 128>("cta_group::2 M=128");
  return 0;
}
