// Experiment: tensor-pipe cost of tcgen05.cp shapes, alone and interleaved with
// FP4 block-scaled MMAs (M=128,N=256,K=64). One CTA; cycles via clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_19503_b200/csrc/common.cuh"
using namespace realb;

__device__ __forceinline__ void cp_128x256b(uint32_t t, uint64_t d) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t), "l"(d) : "memory");
}
__device__ __forceinline__ void cp_128x128b(uint32_t t, uint64_t d) {
  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(t), "l"(d) : "memory");
}

__global__ void __launch_bounds__(128, 1) kern(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536; i += 128) smem[i] = (uint8_t)(0x22);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t s = smem_u32(smem);
    const uint64_t adesc = umma_desc_sw128(s), bdesc = umma_desc_sw128(s + 16384);
    const uint32_t idesc = idesc_nvfp4(128, 256);
    uint64_t sdesc = 0;
    sdesc |= (uint64_t)(((s + 49152) & 0x3FFFFu) >> 4);
    sdesc |= (uint64_t)(128 >> 4) << 16; sdesc |= (uint64_t)(128 >> 4) << 32; sdesc |= (uint64_t)1 << 46;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) {            // 12 x 32x128b.warpx4
        for (int j = 0; j < 12; ++j) utccp_32x128b_warpx4(tb + 256 + 4 * j, sdesc);
      } else if (mode == 1) {     // 4 MMAs only
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 2) {     // 12 cp + 4 MMA (the current stage)
        for (int j = 0; j < 12; ++j) utccp_32x128b_warpx4(tb + 320 + 4 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 3) {     // 6 x 128x256b
        for (int j = 0; j < 6; ++j) cp_128x256b(tb + 256 + 8 * j, sdesc);
      } else if (mode == 4) {     // 6 x 128x256b + 4 MMA
        for (int j = 0; j < 6; ++j) cp_128x256b(tb + 320 + 8 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 5) {     // 12 x 128x128b
        for (int j = 0; j < 12; ++j) cp_128x128b(tb + 256 + 4 * j, sdesc);
      } else if (mode == 6) {     // 3 x 32x128b.warpx4 + 4 MMA (SFB resident; SFA per MMA... 3 cps)
        for (int j = 0; j < 3; ++j) utccp_32x128b_warpx4(tb + 320 + 4 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 8) {     // 8 cp + 4 MMA (SFA resident)
        for (int j = 0; j < 8; ++j) utccp_32x128b_warpx4(tb + 320 + 4 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 9) {     // 6 cp + 4 MMA
        for (int j = 0; j < 6; ++j) utccp_32x128b_warpx4(tb + 320 + 4 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 10) {    // 4 cp + 4 MMA
        for (int j = 0; j < 4; ++j) utccp_32x128b_warpx4(tb + 320 + 4 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 11) {    // 4 x 128x256b + 4 MMA
        for (int j = 0; j < 4; ++j) cp_128x256b(tb + 320 + 8 * j, sdesc);
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
      } else if (mode == 12) {    // interleaved: (2 cp, 1 mma) x 4
        for (int j = 0; j < 4; ++j) {
          utccp_32x128b_warpx4(tb + 320 + 8 * j, sdesc);
          utccp_32x128b_warpx4(tb + 324 + 8 * j, sdesc);
          umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256, tb + 272, 1);
        }
      } else if (mode == 13) {    // 12 cp + 4 MMA consuming THIS stage's copies (RAW)
        const uint32_t buf = tb + 320 + (r & 1) * 48;
        for (int j = 0; j < 4; ++j) {
          utccp_32x128b_warpx4(buf + 4 * j, sdesc);
          utccp_32x128b_warpx4(buf + 16 + 8 * j, sdesc);
          utccp_32x128b_warpx4(buf + 20 + 8 * j, sdesc);
        }
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, buf + 4 * j, buf + 16 + 8 * j, 1);
      } else if (mode == 14) {    // 12 cp for stage r+1, then 4 MMA consuming stage r (lookahead)
        const uint32_t buf = tb + 320 + (r & 1) * 48, nbuf = tb + 320 + ((r + 1) & 1) * 48;
        for (int j = 0; j < 4; ++j) {
          utccp_32x128b_warpx4(nbuf + 4 * j, sdesc);
          utccp_32x128b_warpx4(nbuf + 16 + 8 * j, sdesc);
          utccp_32x128b_warpx4(nbuf + 20 + 8 * j, sdesc);
        }
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, buf + 4 * j, buf + 16 + 8 * j, 1);
      } else if (mode == 15) {    // 8 cp (SFB only) RAW + 4 MMA, SFA resident
        const uint32_t buf = tb + 384 + (r & 1) * 32;
        for (int j = 0; j < 4; ++j) {
          utccp_32x128b_warpx4(buf + 8 * j, sdesc);
          utccp_32x128b_warpx4(buf + 4 + 8 * j, sdesc);
        }
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, tb + 256 + 4 * j, buf + 8 * j, 1);
      } else if (mode == 16) {    // 12 cp, each reading a different 512 B of a 6 KB stage, + 4 MMA RAW
        const uint32_t buf = tb + 320 + (r & 1) * 48;
        for (int j = 0; j < 12; ++j) utccp_32x128b_warpx4(buf + 4 * j, sdesc + (uint64_t)(j * 32));
        for (int j = 0; j < 4; ++j) umma_nvfp4(tb, adesc + 2 * j, bdesc + 2 * j, idesc, buf + 4 * j, buf + 16 + 8 * j, 1);
      } else if (mode == 7) {     // 4 x bf16 MMA N=256 K=16 (reference rate)
        const uint32_t id16 = idesc_bf16(128, 256);
        for (int j = 0; j < 4; ++j) umma_bf16(tb, adesc + 2 * j, bdesc + 2 * j, id16, 1);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

namespace realb {
void set_error(const char*, ...) {}
int cuda_status(cudaError_t, const char*) { return 0; }
int num_sms() { return 148; }
int make_tmap_2d(CUtensorMap*, CUtensorMapDataType, const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t, CUtensorMapSwizzle) { return 0; }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* names[] = {"12x cp32x128b.warpx4", "4x mma fp4 N256", "12cp+4mma", "6x cp128x256b",
                         "6x cp128x256b+4mma", "12x cp128x128b", "3cp+4mma", "4x mma bf16 N256",
                         "8cp+4mma", "6cp+4mma", "4cp+4mma", "4x cp128x256b+4mma", "(2cp,1mma)x4",
                         "12cp+4mma RAW", "12cp(next)+4mma lookahead", "8cp RAW + 4mma (SFA res)",
                         "12cp spread smem RAW"};
  for (int mode = 0; mode < 17; ++mode) {
    const int reps = 2000;
    kern<<<1, 128, 65536>>>(mode, reps, d);
    kern<<<1, 128, 65536>>>(mode, reps, d);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.1f cycles / rep  (err=%s)\n", names[mode], (double)h / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
