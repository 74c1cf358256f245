// Dev micro-benchmark: dependent random-load latency vs footprint (TLB reach).
// One warp per SM chases a random cyclic permutation spread over `bytes`.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lat_bench.cu -o tools/_bin/lat_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>

__global__ void chase(const uint64_t* __restrict__ next, uint64_t start, int steps, unsigned long long* out, uint64_t stride) {
  uint64_t i = (start + blockIdx.x * 7919ULL * stride) % (1ULL << 62);
  const unsigned long long t0 = clock64();
  uint64_t x = i;
  for (int k = 0; k < steps; ++k) x = __ldcg(next + x);
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / steps + (x == 12345678901ULL);
}

int main(int argc, char** argv) {
  const int blocks = argc > 1 ? atoi(argv[1]) : 1;
  for (double gb : {0.0625, 0.25, 1.0, 4.0, 16.0, 64.0}) {
    const uint64_t bytes = static_cast<uint64_t>(gb * (1ULL << 30));
    // one chase node per 4 KB "line group": a random cycle over nodes spaced 4 KB apart
    const uint64_t spacing = 4096 / 8;  // in uint64 elements
    const uint64_t nodes = bytes / 4096;
    uint64_t* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) { printf("%.3f GB: alloc failed\n", gb); continue; }
    std::vector<uint64_t> perm(nodes);
    for (uint64_t k = 0; k < nodes; ++k) perm[k] = k;
    std::mt19937_64 rng(7);
    for (uint64_t k = nodes - 1; k > 0; --k) std::swap(perm[k], perm[rng() % (k + 1)]);
    std::vector<uint64_t> h(nodes);
    // write next pointers node-by-node via a staging buffer of (index,value) pairs
    std::vector<uint64_t> idx(nodes), val(nodes);
    for (uint64_t k = 0; k < nodes; ++k) {
      idx[k] = perm[k] * spacing;
      val[k] = perm[(k + 1) % nodes] * spacing;
    }
    // host copy of the sparse array is too big for 64 GB; scatter on device
    uint64_t *di, *dv;
    cudaMalloc(&di, nodes * 8);
    cudaMalloc(&dv, nodes * 8);
    cudaMemcpy(di, idx.data(), nodes * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, val.data(), nodes * 8, cudaMemcpyHostToDevice);
    // tiny scatter kernel via thrust-free lambda: use a generic kernel below
    extern __global__ void scatter(uint64_t*, const uint64_t*, const uint64_t*, uint64_t);
    scatter<<<(nodes + 255) / 256, 256>>>(d, di, dv, nodes);
    cudaDeviceSynchronize();
    unsigned long long* out;
    cudaMalloc(&out, blocks * 8);
    chase<<<blocks, 1>>>(d, perm[0] * spacing, 2000, out, spacing);
    chase<<<blocks, 1>>>(d, perm[0] * spacing, 20000, out, spacing);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> o(blocks);
    cudaMemcpy(o.data(), out, blocks * 8, cudaMemcpyDeviceToHost);
    unsigned long long s = 0;
    for (auto v : o) s += v;
    printf("footprint %7.3f GB  nodes %9llu  blocks %d  cycles per dependent load %llu  (%s)\n", gb,
           (unsigned long long)nodes, blocks, s / blocks, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(di); cudaFree(dv); cudaFree(out);
  }
  return 0;
}
__global__ void scatter(uint64_t* d, const uint64_t* i, const uint64_t* v, uint64_t n) {
  const uint64_t k = blockIdx.x * 256ULL + threadIdx.x;
  if (k < n) d[i[k]] = v[k];
}
