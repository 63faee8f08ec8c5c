// K1 on CTA pairs (tcgen05 cta_group::2), BF16, for nets whose weights do not
// fit one SM (BASELINE cfg 3: 14-256-256-256-1, 264 KB of BF16 weights).
//
// A cluster of two CTAs sweeps 256-row tiles: CTA rank r owns rows
// [128 r, 128 r + 128) of every tile in its own TMEM (D: H fp32 columns, A:
// H/2 packed bf16 columns, A0 and a ones block) and holds, in shared memory,
// columns [r H/2, (r+1) H/2) of every layer's B operand (+ its bias K block) —
// 140 KB per SM for cfg 3.  The leader CTA (rank 0) issues every
// tcgen05.mma.cta_group::2 (M = 256, N = H, A from TMEM) after the eight (x NSUB)
// warps of both CTAs have arrived on its "A ready" mbarrier (the peer's warps
// arrive remotely, release at cluster scope), and commits each layer to the
// "D ready" mbarrier of both CTAs (multicast).  Epilogues and the final FP32
// layer are CTA-local: a row's H columns live in its own CTA's TMEM.  Columns
// of an epilogue are split over NSUB warpgroups; the next tile's layer 1 is
// released as soon as the final layer's TMEM loads are done.
#pragma once
#include "sweep_kernel.cuh"

namespace surr {

template <int H>
struct CfgPair {
  static constexpr int NSUB = H >= 256 ? 2 : 1;         // warpgroups per CTA (split columns)
  static constexpr int CPS = H / NSUB;                  // columns per sub
  static constexpr int A_COL = H;                       // A operand: H/2 packed columns
  static constexpr int A0_COL = H + H / 2;              // layer-1 operand (8 columns)
  static constexpr int ONES_COL = A0_COL + 8;           // bias K block operand
  static constexpr int NEED = ONES_COL + 8;
  static constexpr int TMEM_COLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 * NSUB;
  static_assert(NEED <= 512, "TMEM budget");
};

template <int H, int SPG>
__global__ void __launch_bounds__(CfgPair<H>::THREADS, 1)
    sweep_kernel_pair(const __grid_constant__ KParams p, int mode) {
  using C = CfgPair<H>;
  constexpr int NG = K0 / SPG;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);  // [0] load, [1] A ready (leader), [2] D ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  float* red = reinterpret_cast<float*>(smem + p.smem_a0);           // [sub][row] partials
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup (both CTAs)
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 4 * C::NSUB * 2);  // every warp of both CTAs
      mbar_init(&bars[2], 1);                // multicast commit from the leader
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint8_t* wsrc = (const uint8_t*)p.w_gmem + (size_t)rank * p.w_rank_stride;
      const uint32_t total = p.w_bytes + (mode == MODE_PREDICT ? 0u : p.lut_bytes);
      mbar_arrive_expect_tx(&bars[0], total);
      for (uint32_t off = 0; off < p.w_bytes; off += 32768u)
        bulk_g2s(smem + off, wsrc + off, min(32768u, p.w_bytes - off), &bars[0]);
      if (mode != MODE_PREDICT && p.lut_bytes) bulk_g2s(smem + p.smem_lut, p.lut_gmem, p.lut_bytes, &bars[0]);
    }
    __syncwarp();
    tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  } else if (warp == 1 && mode == MODE_TOPK) {
    for (uint32_t i = lane; i < p.k; i += 32) {
      ts.lists[i].idx = IDX_SENT;
      ts.lists[i].key = KEY_SENT;
      ts.lists[i].pad = 0;
    }
    if (lane == 0) {
      ts.misc[0] = 0; ts.misc[1] = 0; ts.misc[2] = KEY_SENT; ts.misc[3] = 0xFFFFFFFFu; ts.misc[4] = 0xFFFFFFFFu;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t q = warp >> 2;          // sub (column split)
  const bool first = q == 0, last = q == C::NSUB - 1;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t tl = (wq * 32u) << 16;
  const uint32_t dcol = tmem_base + tl + q * C::CPS;
  const uint32_t acol = tmem_base + tl + C::A_COL;
  const uint32_t a0col = tmem_base + tl + C::A0_COL;
  if (first) {  // constant ones block of the bias K step (each CTA's 128 lanes)
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = 0x00003F80u;
    tmem_st8(tmem_base + tl + C::ONES_COL, ones);
    tmem_wait_st();
  }
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)wq * CAND_CAP;
  uint32_t ncand = 0;
  const bool issuer = leader && warp == 0;
  const uint32_t sb = smem_u32(smem);
  const uint32_t idesc = p.idesc;  // M = 256, N = H
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint32_t npairs = gridDim.x / 2;
  const uint64_t pair = blockIdx.x / 2;
  uint32_t pha = 0, phd = 0;

  // every warp of both CTAs -> leader's "A ready"; the leader's issuer waits and
  // issues layer l's UMMA chain for the 256-row tile
  auto arrive_and_issue = [&](uint32_t l) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_cluster(&bars[1], 0);
    if (issuer) {
      mbar_wait_cluster(&bars[1], pha);
      tc_fence_after();
      if (elect_one()) {
        if (l == 0) {
          umma_f16_ts_pair(tmem_base, tmem_base + C::A0_COL, d_b1, idesc, 0u);
        } else {
          const uint64_t db = make_bdesc(sb + p.off_bh + (l - 1) * p.stride_bh, p.sbo_bh);
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk)
            umma_f16_ts_pair(tmem_base, tmem_base + C::A_COL + kk * 8, db + kk * 16, idesc, kk > 0);
          umma_f16_ts_pair(tmem_base, tmem_base + C::ONES_COL, db + (H / 16) * 16, idesc, 1u);
        }
        umma_commit_pair(&bars[2]);
      }
      __syncwarp();
    }
    pha ^= 1u;
  };

  uint64_t tile = pair;
  uint64_t I = p.begin + tile * (2 * TILE_M) + rank * TILE_M + row;
  const uint64_t dI = (uint64_t)npairs * 2 * TILE_M;
  uint32_t D[MAXG];
  if (first && mode != MODE_PREDICT) init_digits_n<NG>(p.R, I, D);
  mbar_wait(&bars[0], 0);

  A0Regs a0;
  if (tile < p.num_tiles) {
    if (first) {
      if (mode == MODE_PREDICT) make_a0_predict<PREC_BF16>(p, I < p.end ? I : p.begin, a0);
      else if (SPG == 4) make_a0_sweep4(p, slut, D, a0);
      else make_a0_sweep<PREC_BF16>(p, slut, D, a0);
      tmem_st8(a0col, a0.hi);
      tmem_wait_st();
    }
    arrive_and_issue(0);
  }
  for (; tile < p.num_tiles; tile += npairs) {
    const bool valid = I < p.end;
    const uint64_t In = I + dI;
    const bool has_next = tile + npairs < p.num_tiles;
    float part = 0.0f;
    for (uint32_t l = 0; l < p.NL; ++l) {
      if (l + 1 == p.NL && p.NL > 1 && first && has_next) {  // next tile's A0 while the last layer runs
        if (mode == MODE_PREDICT) {
          make_a0_predict<PREC_BF16>(p, In < p.end ? In : p.begin, a0);
        } else {
          odometer_step_n<NG>(p.R, p.dD, D);
          if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC_BF16>(p, slut, D, a0);
        }
        tmem_st8(a0col, a0.hi);
      }
      mbar_wait(&bars[2], phd);
      phd ^= 1u;
      tc_fence_after();
      if (l + 1 < p.NL) {
        // hidden epilogue: this sub's columns -> packed bf16 A (bias already in D)
#pragma unroll
        for (int c = 0; c < C::CPS / 32; c += 2) {
          uint32_t v[2][32];
          tmem_ld32(dcol + c * 32, v[0]);
          if (C::CPS / 32 > 1) tmem_ld32(dcol + (c + 1) * 32, v[1]);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && C::CPS / 32 == 1) break;
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              pk[j] = relu_bf16x2(__uint_as_float(v[u][2 * j]), __uint_as_float(v[u][2 * j + 1]));
            tmem_st16(acol + (q * C::CPS + (c + u) * 32) / 2, pk);
          }
        }
        tmem_wait_st();
        arrive_and_issue(l + 1);
      } else {
        if (p.NL == 1 && first && has_next) {  // single hidden layer: L1 (reads A0) is done only now
          if (mode == MODE_PREDICT) {
            make_a0_predict<PREC_BF16>(p, In < p.end ? In : p.begin, a0);
          } else {
            odometer_step_n<NG>(p.R, p.dD, D);
            if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC_BF16>(p, slut, D, a0);
          }
          tmem_st8(a0col, a0.hi);
        }
        // final FP32 layer over this sub's columns: w relu(x) = (w/2) x + (w/2) |x|,
        // w' in shared memory (broadcast loads); release D to the next tile first
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        const float4* w4 = reinterpret_cast<const float4*>(smem + p.off_fin) + q * C::CPS / 4;
#pragma unroll
        for (int c = 0; c < C::CPS / 32; c += 2) {
          uint32_t v[2][32];
          tmem_ld32(dcol + c * 32, v[0]);
          if (C::CPS / 32 > 1) tmem_ld32(dcol + (c + 1) * 32, v[1]);
          tmem_wait_ld();
          if (c + 2 >= C::CPS / 32 && has_next) {
            if (first) tmem_wait_st();   // next A0 stored
            arrive_and_issue(0);         // next tile's layer 1: D fully read
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && C::CPS / 32 == 1) break;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 w = w4[((c + u) * 32 + j) / 4];
              const float x0 = __uint_as_float(v[u][j]), x1 = __uint_as_float(v[u][j + 1]);
              const float x2 = __uint_as_float(v[u][j + 2]), x3 = __uint_as_float(v[u][j + 3]);
              acc[0] = ffma2(pack2(w.x, w.y), pack2(x0, x1), acc[0]);
              acc[1] = ffma2(pack2(w.x, w.y), pack2(fabsf(x0), fabsf(x1)), acc[1]);
              acc[2] = ffma2(pack2(w.z, w.w), pack2(x2, x3), acc[2]);
              acc[3] = ffma2(pack2(w.z, w.w), pack2(fabsf(x2), fabsf(x3)), acc[3]);
            }
          }
        }
        float a8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
        part = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
      }
    }
    float t = part;
    if (C::NSUB > 1) {
      if (!last) red[q * TILE_M + row] = part;
      named_bar_sync(1, 128 * C::NSUB);
      if (last) {
        float sum = 0.0f;
#pragma unroll
        for (int qq = 0; qq + 1 < C::NSUB; ++qq) sum += red[qq * TILE_M + row];
        t = sum + part;
      }
      named_bar_sync(2, 128 * C::NSUB);  // partials consumed before the next tile overwrites them
    }
    if (last) {
      t += p.c_out;
      if (!ens_stage(p, valid, I, t)) {
      } else if (mode == MODE_TOPK) {
        const uint32_t key = f2key(t);
        const bool pass = valid && key <= ts.misc[2];
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, pass);
        if (m) {
          const uint32_t n = __popc(m);
          if (ncand + n > CAND_CAP) {
            lock_acquire(ts, lane);
            warp_merge(ts, mycand, ncand, p.k, lane);
            lock_release(ts, lane);
            ncand = 0;
          }
          if (pass) {
            const uint32_t pos = ncand + __popc(m & ((1u << lane) - 1u));
            mycand[pos].idx = I;
            mycand[pos].key = key;
            mycand[pos].pad = 0;
          }
          ncand += n;
          __syncwarp();
        }
      } else if (valid) {
        p.t_dense[I - p.begin] = t;
      }
    }
    I = In;
  }
  if (last && mode == MODE_TOPK && ncand) {
    lock_acquire(ts, lane);
    warp_merge(ts, mycand, ncand, p.k, lane);
    lock_release(ts, lane);
  }

  // ---- teardown
  tc_fence_before();
  __syncthreads();
  if (mode == MODE_TOPK) {
    const surr_record* L = ts.lists + (size_t)ts.misc[1] * p.k;
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) p.recs[(size_t)blockIdx.x * p.k + i] = L[i];
  }
  cluster_sync();  // the leader's last UMMAs (reading this CTA's TMEM) are complete in both
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace surr
