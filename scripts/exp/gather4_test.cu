// Experiment: TMA tile::gather4 into a SWIZZLE_128B operand tile. Checks that 32
// gather4 loads (4 indexed rows x 64 bf16 each) produce byte-for-byte the smem
// tile a plain 2D tiled load of the pre-gathered rows produces, with which box
// height the tensor map must be encoded, and what out-of-range row indices do
// (zero fill, full complete_tx byte count).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I. scripts/exp/gather4_test.cu \
//        paper_2604_19503_b200/csrc/runtime.cu -lcuda -o /tmp/g4 && /tmp/g4
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cuda_runtime.h>
#include "../../paper_2604_19503_b200/csrc/common.cuh"
using namespace realb;

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__global__ void kern(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap tt,
                     const int* idx, int kb, uint8_t* out_g, uint8_t* out_t, int* status) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(&bar[0], 128 * 128);
  __syncwarp();
  tma_gather4(smem + lane * 512, &tg, &bar[0], kb * 64, idx[4 * lane], idx[4 * lane + 1], idx[4 * lane + 2],
              idx[4 * lane + 3]);
  if (lane == 0) {
    mbar_arrive_expect_tx(&bar[1], 128 * 128);
    tma_load_2d(smem + 16384, &tt, &bar[1], kb * 64, 0);
  }
  // bounded waits: report instead of hanging if the byte count never completes
  for (int b = 0; b < 2; ++b) {
    long long t0 = clock64();
    while (!mbar_test(&bar[b], 0)) {
      if (clock64() - t0 > 2000000000LL) {
        if (lane == 0) status[b] = -1;
        break;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < 16384; i += 32) {
    out_g[i] = smem[i];
    out_t[i] = smem[16384 + i];
  }
}

int main() {
  const int T = 1000, K = 256;
  std::vector<uint16_t> hx((size_t)T * K);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = (uint16_t)(i * 2654435761u >> 7);
  std::vector<int> idx(128);
  srand(1);
  for (int i = 0; i < 128; ++i) idx[i] = rand() % T;
  idx[5] = T;       // out of range rows
  idx[77] = T + 9;
  std::vector<uint16_t> hg((size_t)128 * K, 0);
  for (int i = 0; i < 128; ++i)
    if (idx[i] < T)
      for (int c = 0; c < K; ++c) hg[(size_t)i * K + c] = hx[(size_t)idx[i] * K + c];
  void *dx, *dg, *dog, *dot;
  int *didx, *dst;
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&dg, hg.size() * 2);
  cudaMalloc(&didx, 128 * 4);
  cudaMalloc(&dog, 16384);
  cudaMalloc(&dot, 16384);
  cudaMalloc(&dst, 8);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, hg.data(), hg.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(didx, idx.data(), 128 * 4, cudaMemcpyHostToDevice);
  for (int box_h : {1}) {
    CUtensorMap tg, tt;
    int rc = make_tmap_2d(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dx, K, T, K * 2, 64, box_h,
                          CU_TENSOR_MAP_SWIZZLE_128B);
    int rc2 = make_tmap_2d(&tt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dg, K, 128, K * 2, 64, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
    printf("box_h=%d encode rc=%d rc2=%d %s\n", box_h, rc, rc2, rc ? realb_last_error() : "");
    if (rc || rc2) continue;
    for (int kb = 0; kb < K / 64; ++kb) {
      cudaMemset(dst, 0, 8);
      cudaMemset(dog, 0xEE, 16384);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
      kern<<<1, 32, 40000>>>(tg, tt, didx, kb, (uint8_t*)dog, (uint8_t*)dot, dst);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint8_t> og(16384), ot(16384);
      int st[2];
      cudaMemcpy(og.data(), dog, 16384, cudaMemcpyDeviceToHost);
      cudaMemcpy(ot.data(), dot, 16384, cudaMemcpyDeviceToHost);
      cudaMemcpy(st, dst, 8, cudaMemcpyDeviceToHost);
      int mism = 0, first = -1;
      for (int i = 0; i < 16384; ++i)
        if (og[i] != ot[i]) { if (first < 0) first = i; ++mism; }
      if (mism)  // where does gathered 16-B chunk j sit in the tiled result?
        for (int j = 0; j < 24; ++j) {
          int at = -1;
          for (int q = 0; q < 1024 && at < 0; ++q)
            if (!memcmp(&og[j * 16], &ot[q * 16], 16)) at = q;
          printf("    og chunk %d (row %d piece %d) == ot chunk %d (row %d piece %d)\n", j, j / 8, j % 8, at,
                 at / 8, at % 8);
        }
      printf("  kb=%d err=%s status=%d,%d mismatched bytes=%d first=%d\n", kb, cudaGetErrorString(e), st[0],
             st[1], mism, first);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
