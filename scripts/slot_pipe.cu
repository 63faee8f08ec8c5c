// Microbenchmark (development aid): the MMA / wait / barrier skeleton of the
// 4-slot 16-bit K1 (sweep_kernel8) without its CUDA-core work, to separate the
// tensor pipe's own rate for the phase mix (L1: SS 128x128x16; L2a / L2b: 8 TS
// 128x64x16 + 1 SS 128x64x16) from the per-phase round trip (commit ->
// mbarrier -> wake -> barrier -> issue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o slot_pipe scripts/slot_pipe.cu
// Prints, per variant, cycles per 128-row tile per SM and the tensor-pipe
// utilisation that implies (640 MMA cycles per tile at 4,096 MAC / cycle).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../paper_2306_14011_b200/csrc/sm100_ptx.cuh"

using namespace surr;

__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  return d;
}
__host__ __device__ uint32_t idesc_f16(uint32_t N) {  // F16 A/B, F32 D, K-major, M = 128
  return (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
}

// mode 0: kernel8 skeleton: 4 slots x 4 warps, self-issuing (named barrier, elected lane of warp 0)
// mode 1: same, waits spin on test_wait instead of the suspending try_wait
// mode 2: same as 0 plus the TMEM traffic of the real kernel (epilogue 4 x ld32 + 4 x st16, two 64-column final loads)
// mode 3: one thread issues every phase of every slot back to back (no waits): the MMA mix's own rate
// mode 4: dedicated issuer warp (warp 16): slot warps arrive on a per-slot "ready" mbarrier; the issuer polls all slots
// mode 5: as 4 plus the TMEM traffic of mode 2
__global__ void __launch_bounds__(544, 1) skel(int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[16];
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
      for (int i = 0; i < 4; ++i) mbar_init(&bars[4 + i], 4);  // ready: one arrive per slot warp
      for (int i = 0; i < 4; ++i) mbar_init(&bars[8 + i], 1);  // mode 9: second completion barrier per slot
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc<512>(&tslot);
  }
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tslot;
  const uint32_t sb = smem_u32(smem);
  // weights: W1' 16 x 128 (K-major, SBO 256), W2 halves 144 x 64 (SBO = 144/8*128 = 2304); A0 tiles; ones
  const uint64_t d_b1 = bdesc(sb, 256);
  const uint64_t d_b2a = bdesc(sb + 4096, 2304);
  const uint64_t d_b2b = bdesc(sb + 4096 + 8 * 2304, 2304);
  const uint64_t d_ones = bdesc(sb + 64 * 1024, 256);
  const uint32_t id_full = idesc_f16(128), id_half = idesc_f16(64);
  unsigned long long t0 = clock64();
  auto issue_phase = [&](uint32_t s, int phase) {
    const uint32_t dslot = base + s * 128;
    const uint64_t d_a0 = bdesc(sb + 68 * 1024 + s * 4096, 256);
    if (phase == 0) {
      umma_f16_ss(dslot, d_a0, d_b1, id_full, 0u);
    } else {
      const uint64_t bd = phase == 1 ? d_b2a : d_b2b;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) umma_f16_ts(dslot + 64, dslot + kk * 8, bd + kk * 16, id_half, kk > 0);
      umma_f16_ss(dslot + 64, d_ones, bd + 8 * 16, id_half, 1u);
    }
  };
  auto issue_quarter = [&](uint32_t s, int q) {  // L2 output neurons 32q .. 32q+31 into region 64 + 32 (q & 1)
    const uint32_t dslot = base + s * 128;
    const uint32_t d = dslot + 64 + 32 * (q & 1);
    const uint64_t bd = d_b2a + (uint64_t)q * 64;  // (dummy weight offsets; timing only)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) umma_f16_ts(d, dslot + kk * 8, bd + kk * 16, idesc_f16(32), kk > 0);
    umma_f16_ss(d, d_ones, bd + 8 * 16, idesc_f16(32), 1u);
  };
  auto issue_l2b_part = [&](uint32_t s, int part) {  // L2b output neurons 32 part .. 32 part + 31 -> region 64 + 32 part
    const uint32_t dslot = base + s * 128;
    const uint32_t d = dslot + 64 + 32 * part;
    const uint64_t bd = d_b2b + (uint64_t)part * 64;  // (dummy weight offsets; timing only)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) umma_f16_ts(d, dslot + kk * 8, bd + kk * 16, idesc_f16(32), kk > 0);
    umma_f16_ss(d, d_ones, bd + 8 * 16, idesc_f16(32), 1u);
  };
  // L2 half with the bias put into the accumulator by tcgen05.cp before the 8 TS UMMAs
  // (no ones-block K step): 11 = 16 x 32x128b.warpx4 (512 B of shared memory each, broadcast
  // to the four lane quadrants), 12 = 8 x 128x256b (4 KB each)
  auto issue_half_cp = [&](uint32_t s, int phase, int cpmode) {
    const uint32_t dslot = base + s * 128;
    const uint64_t bd = phase == 1 ? d_b2a : d_b2b;
    if (cpmode == 11) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint64_t sd = bdesc(sb + 80 * 1024 + c * 512, 128);
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dslot + 64 + c * 4), "l"(sd) : "memory");
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint64_t sd = bdesc(sb + 80 * 1024 + (c & 3) * 4096, 256);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(dslot + 64 + c * 8), "l"(sd) : "memory");
      }
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) umma_f16_ts(dslot + 64, dslot + kk * 8, bd + kk * 16, id_half, 1u);
  };
  if ((mode == 11 || mode == 12) && warp < 16) {
    const uint32_t s = warp >> 2, wq = warp & 3;
    const uint32_t dcol = base + s * 128 + ((wq * 32u) << 16);
    uint32_t pa = 0, sink = 0;
    auto sync_issue = [&](auto&& fn) {
      tc_fence_before();
      named_bar_sync(1 + s, 128);
      if (wq == 0) {
        tc_fence_after();
        if (elect_one()) fn();
        __syncwarp();
      }
    };
    auto waitA = [&]() { mbar_wait(&bars[s], pa); pa ^= 1u; tc_fence_after(); };
    auto ld64 = [&](uint32_t col) { uint32_t v[2][32]; tmem_ld32(col, v[0]); tmem_ld32(col + 32, v[1]); tmem_wait_ld(); sink += v[0][3] + v[1][17]; };
    sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    for (int it = 0; it < iters; ++it) {
      waitA();  // L1
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        uint32_t v[2][32];
        tmem_ld32(dcol + c * 32, v[0]);
        tmem_ld32(dcol + (c + 1) * 32, v[1]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = v[u][2 * j] ^ v[u][2 * j + 1];
          tmem_st16(dcol + (c + u) * 16, pk);
        }
      }
      tmem_wait_st();
      sync_issue([&] { issue_half_cp(s, 1, mode); umma_commit(&bars[s]); });
      waitA(); ld64(dcol + 64);
      sync_issue([&] { issue_half_cp(s, 2, mode); umma_commit(&bars[s]); });
      waitA(); ld64(dcol + 64);
      if (it + 1 < iters) sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    }
    if (sink == 0x12345678u) out[0] = 0;
  } else if (mode == 10 && warp < 16) {
    // kernel8 skeleton with TMEM traffic, L2b issued as two N = 32 halves: the first as
    // soon as D2a's first 32 columns are in registers, the second after the rest
    const uint32_t s = warp >> 2, wq = warp & 3;
    const uint32_t dcol = base + s * 128 + ((wq * 32u) << 16);
    uint32_t pa = 0, pb = 0, sink = 0;
    auto sync_issue = [&](auto&& fn) {
      tc_fence_before();
      named_bar_sync(1 + s, 128);
      if (wq == 0) {
        tc_fence_after();
        if (elect_one()) fn();
        __syncwarp();
      }
    };
    auto waitA = [&]() { mbar_wait(&bars[s], pa); pa ^= 1u; tc_fence_after(); };
    auto waitB = [&]() { mbar_wait(&bars[8 + s], pb); pb ^= 1u; tc_fence_after(); };
    auto ld32 = [&](uint32_t col) { uint32_t v[32]; tmem_ld32(col, v); tmem_wait_ld(); sink += v[3] + v[17]; };
    sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    for (int it = 0; it < iters; ++it) {
      waitA();  // L1
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        uint32_t v[2][32];
        tmem_ld32(dcol + c * 32, v[0]);
        tmem_ld32(dcol + (c + 1) * 32, v[1]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = v[u][2 * j] ^ v[u][2 * j + 1];
          tmem_st16(dcol + (c + u) * 16, pk);
        }
      }
      tmem_wait_st();
      sync_issue([&] { issue_phase(s, 1); umma_commit(&bars[s]); });
      waitA();  // L2a
      ld32(dcol + 64);
      sync_issue([&] { issue_l2b_part(s, 0); umma_commit(&bars[s]); });
      ld32(dcol + 96);
      sync_issue([&] { issue_l2b_part(s, 1); umma_commit(&bars[8 + s]); });
      waitA(); ld32(dcol + 64);
      waitB(); ld32(dcol + 96);
      if (it + 1 < iters) sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    }
    if (sink == 0x12345678u) out[0] = 0;
  } else if (mode == 9 && warp < 16) {
    // L2 in four N = 32 quarters alternating between two 32-column regions, so each
    // quarter's final load overlaps the next quarter's UMMAs (TMEM traffic included)
    const uint32_t s = warp >> 2, wq = warp & 3;
    const uint32_t dcol = base + s * 128 + ((wq * 32u) << 16);
    uint32_t pa = 0, pb = 0, sink = 0;
    auto sync_issue = [&](auto&& fn) {
      tc_fence_before();
      named_bar_sync(1 + s, 128);
      if (wq == 0) {
        tc_fence_after();
        if (elect_one()) fn();
        __syncwarp();
      }
    };
    auto waitA = [&]() { mbar_wait(&bars[s], pa); pa ^= 1u; tc_fence_after(); };
    auto waitB = [&]() { mbar_wait(&bars[8 + s], pb); pb ^= 1u; tc_fence_after(); };
    auto ld32 = [&](uint32_t col) { uint32_t v[32]; tmem_ld32(col, v); tmem_wait_ld(); sink += v[3] + v[17]; };
    sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    for (int it = 0; it < iters; ++it) {
      waitA();  // L1
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        uint32_t v[2][32];
        tmem_ld32(dcol + c * 32, v[0]);
        tmem_ld32(dcol + (c + 1) * 32, v[1]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = v[u][2 * j] ^ v[u][2 * j + 1];
          tmem_st16(dcol + (c + u) * 16, pk);
        }
      }
      tmem_wait_st();
      sync_issue([&] { issue_quarter(s, 0); umma_commit(&bars[s]); issue_quarter(s, 1); umma_commit(&bars[8 + s]); });
      waitA(); ld32(dcol + 64);
      sync_issue([&] { issue_quarter(s, 2); umma_commit(&bars[s]); });
      waitB(); ld32(dcol + 96);
      sync_issue([&] { issue_quarter(s, 3); umma_commit(&bars[8 + s]); });
      waitA(); ld32(dcol + 64);
      waitB(); ld32(dcol + 96);
      if (it + 1 < iters) sync_issue([&] { issue_phase(s, 0); umma_commit(&bars[s]); });
    }
    if (sink == 0x12345678u) out[0] = 0;
  } else if (mode == 3) {
    if (threadIdx.x == 0) {
      for (int it = 0; it < iters; ++it)
        for (int ph = 0; ph < 3; ++ph)
          for (uint32_t s = 0; s < 4; ++s) issue_phase(s, ph);
      umma_commit(&bars[0]);
      mbar_wait(&bars[0], 0);
    }
  } else if (warp < 16) {
    const uint32_t s = warp >> 2, wq = warp & 3;
    const uint32_t dcol = base + s * 128 + ((wq * 32u) << 16);
    // 6: epilogue ld/st only; 7: final loads only; 8: all traffic issued after the next phase (off the chain)
    const bool epi_t = mode == 2 || mode == 5 || mode == 6;
    const bool fin_t = mode == 2 || mode == 5 || mode == 7;
    const bool late = mode == 8;
    const bool central = mode == 4 || mode == 5;
    uint32_t ph = 0;
    auto wait_done = [&]() {
      if (mode == 1) { while (!mbar_test(&bars[s], ph)) {} }
      else mbar_wait(&bars[s], ph);
      ph ^= 1u;
      tc_fence_after();
    };
    auto go = [&](int phase) {
      tc_fence_before();
      if (central) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[4 + s]);
        return;
      }
      named_bar_sync(1 + s, 128);
      if (wq == 0) {
        tc_fence_after();
        if (elect_one()) {
          issue_phase(s, phase);
          umma_commit(&bars[s]);
        }
        __syncwarp();
      }
    };
    uint32_t sink = 0;
    if (!central) go(0);
    else go(0);
    for (int it = 0; it < iters; ++it) {
      wait_done();  // L1
      if (late) go(1);
      if (epi_t || late) {
#pragma unroll
        for (int c = 0; c < 4; c += 2) {
          uint32_t v[2][32];
          tmem_ld32(dcol + c * 32, v[0]);
          tmem_ld32(dcol + (c + 1) * 32, v[1]);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = v[u][2 * j] ^ v[u][2 * j + 1];
            tmem_st16(dcol + (c + u) * 16, pk);
          }
        }
        tmem_wait_st();
      }
      if (!late) go(1);
      wait_done();  // L2a
      if (late) go(2);
      if (fin_t || late) {
        uint32_t v[2][32];
        tmem_ld32(dcol + 64, v[0]);
        tmem_ld32(dcol + 96, v[1]);
        tmem_wait_ld();
        sink += v[0][5] + v[1][3];
      }
      if (!late) go(2);
      wait_done();  // L2b
      if (late && it + 1 < iters) go(0);
      if (fin_t || late) {
        uint32_t v[2][32];
        tmem_ld32(dcol + 64, v[0]);
        tmem_ld32(dcol + 96, v[1]);
        tmem_wait_ld();
        sink += v[0][7] + v[1][9];
      }
      if (!late && it + 1 < iters) go(0);
    }
    if (sink == 0x12345678u) out[0] = 0;
  } else if (warp == 16 && (mode == 4 || mode == 5)) {
    // dedicated issuer: slot s is ready for its next phase when its four warps arrived
    int next[4] = {0, 0, 0, 0};
    uint32_t rph[4] = {0, 0, 0, 0};
    int issued[4] = {0, 0, 0, 0};
    const int total = 3 * iters;  // phases per slot (the first L1 included, the last tile's L1 not issued)
    int remaining = 4 * (3 * iters - 0);
    // per slot the phases are L1, L2a, L2b, L1, ... ; the last go(0) is skipped by the slot warps
    remaining = 4 * (3 * (iters - 1) + 3);
    while (remaining > 0) {
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) {
        if (issued[s] < total && mbar_test(&bars[4 + s], rph[s])) {
          rph[s] ^= 1u;
          tc_fence_after();
          if (elect_one()) {
            issue_phase(s, next[s]);
            umma_commit(&bars[s]);
          }
          __syncwarp();
          next[s] = next[s] == 2 ? 0 : next[s] + 1;
          ++issued[s];
          --remaining;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = (unsigned long long)iters * 4;  // tiles
  }
  if (warp == 0) { tc_fence_after(); tmem_dealloc(base, 512); }
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d;
  cudaFuncSetAttribute(skel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaMalloc(&d, 148 * 2 * 8);
  std::vector<unsigned long long> h(148 * 2);
  const char* names[] = {"kernel8 skeleton (try_wait, named barrier, self-issue)", "same, spin test_wait",
                         "skeleton + TMEM traffic (epilogue ld/st, final loads)", "one thread, no waits (MMA mix rate)",
                         "dedicated issuer warp polling slots", "dedicated issuer + TMEM traffic",
                         "skeleton + epilogue ld/st only", "skeleton + final loads only",
                         "skeleton + all TMEM traffic off the chain (after the next issue)",
                         "L2 as four N=32 quarters in two alternating regions, with TMEM traffic",
                         "TMEM traffic, L2b as two N=32 halves issued as D2a's halves are loaded",
                         "TMEM traffic, L2 bias by tcgen05.cp 32x128b.warpx4 x16 (no ones K step)",
                         "TMEM traffic, L2 bias by tcgen05.cp 128x256b x8 (no ones K step)"};
  std::vector<int> modes;
  for (int i = 1; i < argc; ++i) modes.push_back(atoi(argv[i]));
  if (modes.empty()) modes = {0, 2, 6, 7};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode : modes) {
      const int iters = 2000;
      const int threads = (mode == 4 || mode == 5) ? 544 : 512;
      skel<<<148, threads, 100 * 1024>>>(mode, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d error %s\n", mode, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h.data(), d, 148 * 2 * 8, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int b = 0; b < 148; ++b) cyc += (double)h[b * 2] / h[b * 2 + 1];
      cyc /= 148;
      printf("mode %d %-58s %8.1f cycles / tile  -> tensor pipe %.3f of 640\n", mode, names[mode], cyc, 640.0 / cyc);
    }
  return 0;
}
