// Microbenchmark (development aid): tcgen05.ld / tcgen05.st throughput per SM
// for the shapes an epilogue can use.  nwarps warps (multiple of 4), each
// loading `cols` 32-bit columns of its lane quadrant per iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_rate scripts/tmem_rate.cu
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2306_14011_b200/csrc/sm100_ptx.cuh"

using namespace surr;

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%"
      "18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld_32x32b_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%"
      "18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,"
      "%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

// mode 0: 32x32b.x32 loads (4 KB per warp-instruction), wait after each
// mode 1: 32x32b.x32 x2 then wait
// mode 2: 16x256b.x8 (16 lanes x 8 x 256b = 4 KB), wait after each
// mode 3: 32x32b.x64 (8 KB), wait after each
// mode 4: 32x32b.x16 stores (2 KB), wait after each
__global__ void bench(int mode, int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tslot + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 64;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      uint32_t v[32];
      tmem_ld32(base + (it & 1) * 32, v);
      tmem_wait_ld();
      acc += v[0] ^ v[31];
    } else if (mode == 1) {
      uint32_t v[32], w[32];
      tmem_ld32(base, v);
      tmem_ld32(base + 32, w);
      tmem_wait_ld();
      acc += v[0] ^ w[31];
    } else if (mode == 2) {
      uint32_t v[32];
      ld_16x256b_x8(base + (it & 1) * 32, v);
      tmem_wait_ld();
      acc += v[0] ^ v[31];
    } else if (mode == 3) {
      uint32_t v[64];
      ld_32x32b_x64(base, v);
      tmem_wait_ld();
      acc += v[0] ^ v[63];
    } else {
      uint32_t v[16];
      for (int j = 0; j < 16; ++j) v[j] = it + j;
      tmem_st16(base + (it & 3) * 16, v);
      tmem_wait_st();
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  std::vector<unsigned long long> h(148);
  const char* names[] = {"32x32b.x32 ld", "32x32b.x32 ld x2", "16x256b.x8 ld", "32x32b.x64 ld", "32x32b.x16 st"};
  const double bytes_per_warp[] = {4096, 8192, 4096, 8192, 2048};
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode)
    for (int nw : {4, 8, 12, 16}) {
      bench<<<148, nw * 32>>>(mode, iters, d, sink);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int b = 0; b < 148; ++b) cyc += h[b];
      cyc /= 148;
      printf("%-18s warps %2d: %7.1f cycles/iter, %6.1f B/clk/SM\n", names[mode], nw, cyc / iters,
             bytes_per_warp[mode] * nw * iters / cyc);
    }
  return 0;
}
