// Dev micro-benchmark of flat_sweep (bc_flat.cuh) alone: one warp per CTA
// sweeps the same source (data from tools/sweep_data.py); prints the depth
// and cycles per level.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -std=c++20 -I paper_1701_05975_b200/csrc tools/sweep_bench.cu -o tools/_bin/sweep_bench
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bc_flat.cuh"

using namespace wbc_dev;

namespace wbc_dev {
template <int KE>
__device__ __forceinline__ uint32_t flat_sweep_b(const uint32_t* __restrict__ ord_d, const uint32_t* __restrict__ ent,
                                              uint32_t reached, uint32_t B, uint32_t* bucket, uint32_t* s_sd,
                                              uint32_t* s_en, uint32_t lane) {
  const uint32_t M = B - 1;
  constexpr uint32_t kRingPos = kFlatRing * kFlatChunk;
  static_assert(kFlatChunk >= 64, "a 64-position block spans at most two chunks");
  for (uint32_t i = lane; i < B; i += 32) bucket[i] = 0;
  auto stage = [&](uint32_t c) {  // chunk c -> ring slot c % kFlatRing
    if (c * kFlatChunk < reached) {
      const uint32_t sl = c % kFlatRing;
      for (uint32_t k = lane; k < kFlatChunk / 4; k += 32)
        cp_async16(s_sd + sl * kFlatChunk + 4 * k, ord_d + c * kFlatChunk + 4 * k);
      for (uint32_t k = lane; k < kFlatChunk * KE / 4; k += 32)
        cp_async16(s_en + sl * kFlatChunk * KE + 4 * k,
                   ent + static_cast<uint64_t>(c) * kFlatChunk * KE + 4 * k);
    }
    cp_async_commit();
  };
  // chunks [cur, cur + kFlatRing) are issued; cur and cur + 1 are complete
  uint32_t issued = 0, cur = 0;
  for (; issued < static_cast<uint32_t>(kFlatRing); ++issued) stage(issued);
  cp_async_wait<kFlatRing - 2>();
  __syncwarp();
  auto advance_to = [&](uint32_t q) {  // position q (only grows) moves the window
    while (cur < q / kFlatChunk) {
      __syncwarp();  // every lane is done with chunk cur's slot
      ++cur;
      stage(issued++);
      cp_async_wait<kFlatRing - 2>();
      __syncwarp();
    }
  };
  // level 0 = {s}: insert its entries (d(s) = 0)
  uint32_t newmin = kInfDist;  // smallest key inserted by the last level, live at its threshold
  if (lane < KE) {
    const uint32_t e = s_en[lane];
    if (e) {
      atomicMax(bucket + ((e & 0xFFFFu) & M), (e >> 16) + 1);
      newmin = e & 0xFFFFu;  // d(v) = e >> 16 >= 1 = tau: live
    }
  }
  newmin = __reduce_min_sync(0xffffffffu, newmin);
  __syncwarp();
  uint32_t tau = 1, pos = 1, levels = 1;
  for (;;) {
    // the next threshold: the first live key > tau in the ring, or newmin
    uint32_t nxt = newmin;
    for (uint32_t base = tau + 1; base < tau + B && base <= nxt; base += 32) {
      const uint32_t k = base + lane;
      const bool live = k < tau + B && bucket[k & M] >= tau + 1;
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (m) {
        nxt = min(nxt, base + __ffs(m) - 1);
        break;
      }
    }
    if (nxt == kInfDist) break;
    // the new level: positions [pos, end) with d < nxt, 32 per step
    uint32_t q = pos, lmin = kInfDist;
    while (q < reached) {
      advance_to(q);
      const uint32_t qq = q + lane;
      const bool ok = qq < reached;
      const uint32_t d = ok ? s_sd[qq % kRingPos] : kInfDist;
      const uint4 e4 = *reinterpret_cast<const uint4*>(s_en + (qq % kRingPos) * KE);
      const bool in = ok && d < nxt;
      const uint32_t got = __popc(__ballot_sync(0xffffffffu, in));
      const uint32_t ex[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t dvp1 = d + (ex[x] >> 16) + 1;
        const uint32_t key = d + (ex[x] & 0xFFFFu);
        const bool v = in && ex[x] != 0u && dvp1 > nxt;
        atomicMax(bucket + (key & M), v ? dvp1 : 0u);  // unconditional: no branch per entry
        lmin = v ? min(lmin, key) : lmin;
      }
      q += got;
      if (got < 32) break;
    }
    newmin = __reduce_min_sync(0xffffffffu, lmin);
    __syncwarp();  // this level's inserts are visible to the scans after the next one
    pos = q;
    tau = nxt;
    ++levels;

  }
  cp_async_wait<0>();
  __syncwarp();
  return levels;
}

}  // namespace wbc_dev


template <int V>
__global__ void sweep_kernel(const uint32_t* ord_d, const uint32_t* ent, uint32_t reached, uint32_t B,
                             uint32_t* levels_out, unsigned long long* cycles_out) {
  extern __shared__ uint32_t sm[];
  uint32_t* bucket = sm;
  uint32_t* s_sd = bucket + B;
  uint32_t* s_en = s_sd + kFlatRing * kFlatChunk;
  const unsigned long long t0 = clock64();
  const uint32_t lv = V == 0   ? flat_sweep<4>(ord_d, ent, reached, B, bucket, s_sd, s_en, threadIdx.x & 31)
                      : V == 1 ? flat_sweep_b<4>(ord_d, ent, reached, B, bucket, s_sd, s_en, threadIdx.x & 31)
                               : flat_sweep<4>(ord_d, ent, reached, B, bucket, s_sd, s_en, threadIdx.x & 31);
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    levels_out[blockIdx.x] = lv;
    cycles_out[blockIdx.x] = t1 - t0;
  }
}

int main(int argc, char** argv) {
  const char* dir = argc > 1 ? argv[1] : "gpurun_out/sweep";
  const int ctas = argc > 2 ? atoi(argv[2]) : 1;
  char path[512];
  snprintf(path, sizeof path, "%s/meta.txt", dir);
  FILE* f = fopen(path, "r");
  unsigned reached = 0, B = 0, want = 0;
  if (!f || fscanf(f, "%u %u %u", &reached, &B, &want) != 3) return 1;
  fclose(f);
  const size_t cap = (reached + kFlatChunk * 2) / kFlatChunk * kFlatChunk + kFlatChunk;
  std::vector<uint32_t> od(cap, 0xFFFFFFFFu), en(cap * 4, 0);
  snprintf(path, sizeof path, "%s/ord_d.bin", dir);
  f = fopen(path, "rb");
  if (fread(od.data(), 4, reached, f) != reached) return 2;
  fclose(f);
  snprintf(path, sizeof path, "%s/ent.bin", dir);
  f = fopen(path, "rb");
  if (fread(en.data(), 4, size_t{reached} * 4, f) != size_t{reached} * 4) return 3;
  fclose(f);
  uint32_t *d_od, *d_en, *d_lv;
  unsigned long long* d_cy;
  cudaMalloc(&d_od, od.size() * 4);
  cudaMalloc(&d_en, en.size() * 4);
  cudaMalloc(&d_lv, ctas * 4);
  cudaMalloc(&d_cy, ctas * 8);
  cudaMemcpy(d_od, od.data(), od.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_en, en.data(), en.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (B + kFlatRing * kFlatChunk * 5) * 4;
  cudaFuncSetAttribute(sweep_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sweep_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sweep_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 6; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    if (rep < 2)
      sweep_kernel<0><<<ctas, 32, smem>>>(d_od, d_en, reached, B, d_lv, d_cy);
    else if (rep < 4)
      sweep_kernel<1><<<ctas, 32, smem>>>(d_od, d_en, reached, B, d_lv, d_cy);
    else
      sweep_kernel<2><<<ctas, 32, smem>>>(d_od, d_en, reached, B, d_lv, d_cy);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<uint32_t> lv(ctas);
    std::vector<unsigned long long> cy(ctas);
    cudaMemcpy(lv.data(), d_lv, ctas * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cy.data(), d_cy, ctas * 8, cudaMemcpyDeviceToHost);
    printf("v%d ctas=%d levels=%u (want %u) %s  cycles=%llu  cycles/level=%.0f  wall %.2f ms  err=%s\n", rep / 2, ctas, lv[0], want,
           lv[0] == want ? "OK" : "MISMATCH", cy[0], double(cy[0]) / lv[0], ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
