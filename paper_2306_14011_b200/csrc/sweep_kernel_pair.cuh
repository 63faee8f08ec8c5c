// K1 on CTA pairs (tcgen05 cta_group::2), BF16, for nets whose weights do not
// fit one SM (BASELINE cfg 3: 14-256-256-256-1, 264 KB of BF16 weights).
//
// A cluster of two CTAs sweeps 256-row tiles: CTA rank r owns rows
// [128 r, 128 r + 128) of every tile (its TMEM lanes) and holds, in shared
// memory, 64 of the 128 output columns of each N-half of every layer's B
// operand (+ its bias K block): 140 KB per SM for cfg 3.  The leader CTA's
// issuer warp runs every tcgen05.mma.cta_group::2 (M = 256, N = H/2 per half).
//
// TMEM (512 columns) is two H-column regions used alternately by consecutive
// layers.  A hidden epilogue writes its packed bf16 A IN PLACE over the region
// it reads (chunk c is read before columns 16c.. are written), so layer l+1
// reads A from one region while writing D into the other.  Every layer is
// issued as two N-halves (own commit each) and streamed in K quarters:
//   sub q (warps 4q .. 4q+3 of each CTA) owns output columns [q H/2, (q+1) H/2);
//   it signals "A quarter 2q+j ready" after packing its j-th quarter, and the
//   issuer runs those K-steps of the next layer for both N-halves right away,
// so the epilogue of half a overlaps the MMA of half b and the epilogues
// overlap the next layer's first K-steps.  The layer-1 operand A0 and the
// bias "ones" block are SMEM tiles (SS form); a producer warp per CTA decodes
// the next tile's A0 while the hidden layers run.
//
// warps 0-7: epilogue (2 subs x 4), warp 8: A0 producer, warp 9: MMA issuer
// (leader CTA only).  Barriers (leader unless noted): A0F (2 producers), AQ[4]
// (8 warps each), RF (16 warps: previous tile's final layer read its region),
// DA / DB (both CTAs, multicast commits of the N-halves), A0E (both CTAs:
// layer 1 done, A0 tile free).
#pragma once
#include "sweep_kernel3.cuh"  // st_a0_smem, topk_offer

namespace surr {

template <int H, int NS>
struct CfgPair {
  static constexpr int NSUB = NS;          // epilogue warpgroups per CTA (column split)
  static constexpr int HALF = H / 2;       // N per half-MMA
  static constexpr int SUBC = H / NSUB;    // columns per sub
  static constexpr int QC = H / 4;         // columns per K quarter
  static constexpr int QPS = 4 / NSUB;     // quarters per sub
  static constexpr int QSTEPS = QC / 16;   // UMMA K-steps per quarter
  static constexpr int TMEM_COLS = 512;
  static constexpr int EPI_WARPS = 4 * NSUB;
  static constexpr int THREADS = 32 * EPI_WARPS + 64;  // + A0 producer + MMA issuer
  static_assert(2 * H <= 512 && H % 64 == 0, "two H-column regions");
  static_assert(NSUB == 2 || NSUB == 4, "sub count");
};

enum { PB_LOAD = 0, PB_A0F = 1, PB_AQ = 2, PB_RF = 6, PB_DA = 7, PB_DB = 8, PB_A0E = 9 };

template <int H, int SPG, int NS, int PREC = PREC_BF16>
__global__ void __launch_bounds__(CfgPair<H, NS>::THREADS, 1)
    sweep_kernel_pair(const __grid_constant__ KParams p, int mode) {
  using C = CfgPair<H, NS>;
  constexpr int NG = K0 / SPG;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 96);
  uint8_t* a0tile = smem + p.smem_a0;
  float* red = reinterpret_cast<float*>(smem + p.smem_ones + 4096);  // [sub][row] partials of subs < NSUB-1
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup (both CTAs)
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[PB_LOAD], 1);
      mbar_init(&bars[PB_A0F], 2);
      for (int j = 0; j < 4; ++j) mbar_init(&bars[PB_AQ + j], 8);
      mbar_init(&bars[PB_RF], 2 * C::EPI_WARPS);
      mbar_init(&bars[PB_DA], 1);
      mbar_init(&bars[PB_DB], 1);
      mbar_init(&bars[PB_A0E], 1);
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint8_t* wsrc = (const uint8_t*)p.w_gmem + (size_t)rank * p.w_rank_stride;
      const uint32_t total = p.w_bytes + (mode == MODE_PREDICT ? 0u : p.lut_bytes);
      mbar_arrive_expect_tx(&bars[PB_LOAD], total);
      for (uint32_t off = 0; off < p.w_bytes; off += 32768u)
        bulk_g2s(smem + off, wsrc + off, min(32768u, p.w_bytes - off), &bars[PB_LOAD]);
      if (mode != MODE_PREDICT && p.lut_bytes) bulk_g2s(smem + p.smem_lut, p.lut_gmem, p.lut_bytes, &bars[PB_LOAD]);
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
      ts.misc[0] = 0; ts.misc[1] = 0; ts.misc[2] = KEY_SENT; ts.misc[3] = 0xFFFFFFFFu; ts.misc[4] = 0xFFFFFFFFu; ts.misc[5] = 0;
      for (uint32_t b = 0; b < TOPK_MAX_BUFS; ++b) ts.misc[8 + b] = 0;
    }
  }
  if (warp >= 4 && warp < 8) {  // constant ones tile of the bias K step (bf16 1.0 in K slot 0)
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = one16<PREC>();
    st_a0_smem(smem + p.smem_ones, (warp - 4) * 32u + lane, ones);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t npairs = gridDim.x / 2;
  const uint64_t pair = blockIdx.x / 2;
  const uint64_t dI = (uint64_t)npairs * 2 * TILE_M;
  const uint8_t* slut = smem + p.smem_lut;
  mbar_wait(&bars[PB_LOAD], 0);

  if (warp == C::EPI_WARPS + 1) {
    // =========================== MMA issuer (leader) ===========================
    if (leader) {
      const uint32_t sb = smem_u32(smem);
      const uint32_t idesc = p.idesc;  // M = 256, N = H/2
      const uint64_t d_a0 = make_bdesc(sb + p.smem_a0, 256);
      const uint64_t d_ones = make_bdesc(sb + p.smem_ones, 256);
      const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
      const uint64_t b1_half = (8ull * p.sbo_b1) >> 4;  // N-half b: 8 row groups further
      const uint64_t bh_half = (8ull * p.sbo_bh) >> 4;
      uint32_t ph_a0f = 0, ph_rf = 0, ph_db = 0, ph_aq = 0, region = 0, jt = ~0u;  // jt: tile round (trace)
      for (uint64_t tile = pair; tile < p.num_tiles; tile += npairs) {
        // layer 1 (K = 16, A0 from shared memory) into `region`
        if (p.NL == 1 && tile != pair) {  // no hidden GEMM: the final layer's region is rewritten by layer 1
          mbar_wait(&bars[PB_RF], ph_rf);
          ph_rf ^= 1u;
        }
        ++jt;
        mbar_wait(&bars[PB_A0F], ph_a0f);
        ph_a0f ^= 1u;
        tc_fence_after();
        if (lane == 0) trace_ev(p, 0, jt, 0);
        {
          const uint32_t d = tmem_base + region * H;
          if (elect_one()) {
            umma_f16_ss_pair(d, d_a0, d_b1, idesc, 0u);
            umma_commit_pair(&bars[PB_DA]);
            umma_f16_ss_pair(d + C::HALF, d_a0, d_b1 + b1_half, idesc, 0u);
            umma_commit_pair(&bars[PB_DB]);
            umma_commit_pair(&bars[PB_A0E]);
          }
          __syncwarp();
          if (lane == 0) trace_ev(p, 0, jt, 11);
        }
        for (uint32_t l = 1; l < p.NL; ++l) {
          const uint32_t src = tmem_base + region * H;  // packed A of layer l (in place)
          region ^= 1u;
          const uint32_t dst = tmem_base + region * H;
          const uint64_t db = make_bdesc(sb + p.off_bh + (l - 1) * p.stride_bh, p.sbo_bh);
          // NSUB = 2: the previous tile's final layer read `dst` before its subs'
          // AQ arrivals for this layer (sub 0 -> half a, sub 1 -> half b), so no
          // separate wait is needed; with 4 subs half a spans two subs
          if (C::NSUB != 2 && l == 1 && tile != pair) {
            mbar_wait(&bars[PB_RF], ph_rf);
            ph_rf ^= 1u;
          }
          if (lane == 0) trace_ev(p, 0, jt, 1);
          // N-half a streamed over the K quarters as their A columns arrive
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mbar_wait(&bars[PB_AQ + j], ph_aq);
            tc_fence_after();
            if (lane == 0 && l <= 2) trace_ev(p, 0, jt, 2 + (l - 1) * 4 + j);
            if (elect_one()) {
              // quarter j = K [j QC, (j+1) QC): packed A columns of sub j/QPS, chunk j%QPS
              const uint32_t acol = src + (j / C::QPS) * C::SUBC + (j % C::QPS) * (C::QC / 2);
#pragma unroll
              for (int s = 0; s < C::QSTEPS; ++s)
                umma_f16_ts_pair(dst, acol + s * 8, db + (j * C::QSTEPS + s) * 16, idesc, (j | s) != 0);
              if (j == 3) {
                umma_f16_ss_pair(dst, d_ones, db + (H / 16) * 16, idesc, 1u);
                umma_commit_pair(&bars[PB_DA]);
              }
            }
            __syncwarp();
          }
          // N-half b in one chain (its output columns belong to the sub whose
          // epilogue starts last; they are rewritten only after its AQ arrivals)
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t acol = src + (j / C::QPS) * C::SUBC + (j % C::QPS) * (C::QC / 2);
#pragma unroll
              for (int s = 0; s < C::QSTEPS; ++s)
                umma_f16_ts_pair(dst + C::HALF, acol + s * 8, db + bh_half + (j * C::QSTEPS + s) * 16, idesc,
                                 (j | s) != 0);
            }
            umma_f16_ss_pair(dst + C::HALF, d_ones, db + bh_half + (H / 16) * 16, idesc, 1u);
            umma_commit_pair(&bars[PB_DB]);
          }
          __syncwarp();
          ph_aq ^= 1u;
        }
        // the last layer (reading the other region as A) completes before the
        // next tile's layer 1 overwrites that region
        ph_db ^= (p.NL - 1) & 1u;  // DB phases of the non-final layers
        if (tile + npairs < p.num_tiles) mbar_wait(&bars[PB_DB], ph_db);
        if (lane == 0) trace_ev(p, 0, jt, 10);
        ph_db ^= 1u;
        region ^= 1u;
      }
    }
  } else if (warp == C::EPI_WARPS) {
    // ============================ A0 producer ============================
    // lane owns rows lane + 32 u (u = 0..3) of this CTA's 128 rows
    uint64_t I0 = p.begin + pair * (2 * TILE_M) + rank * TILE_M + lane;
    uint32_t D[4][MAXG];
    if (mode != MODE_PREDICT) {
#pragma unroll
      for (int u = 0; u < 4; ++u) init_digits_n<NG>(p.R, I0 + 32u * u, D[u]);
    }
    uint32_t ph_e = 0;
    for (uint64_t tile = pair; tile < p.num_tiles; tile += npairs) {
      if (tile != pair) {  // layer 1 of the previous tile has consumed the A0 tile
        mbar_wait(&bars[PB_A0E], ph_e);
        ph_e ^= 1u;
      }
      if (lane == 0) trace_ev(p, 3, (uint32_t)((tile - pair) / npairs), 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        A0Regs a0;
        const uint64_t I = I0 + 32u * u;
        if (mode == MODE_PREDICT) {
          make_a0_predict<PREC>(p, I < p.end ? I : p.begin, a0);
        } else {
          if (tile != pair) odometer_step_n<NG>(p.R, p.dD, D[u]);
          if (SPG == 4) make_a0_sweep4(p, slut, D[u], a0); else make_a0_sweep<PREC>(p, slut, D[u], a0);
          a0_dump<false>(p, mode, a0, I);
        }
        st_a0_smem(a0tile, lane + 32u * u, a0.hi);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&bars[PB_A0F], 0);
      if (lane == 0) trace_ev(p, 3, (uint32_t)((tile - pair) / npairs), 1);
      I0 += dI;
    }
  } else {
    // ============================= epilogue =============================
    const uint32_t q = warp >> 2;  // sub: output columns [q SUBC, (q+1) SUBC)
    const bool last = q == C::NSUB - 1;
    const uint32_t wq = warp & 3u;
    const uint32_t row = wq * 32u + lane;
    const uint32_t tl = (wq * 32u) << 16;
    uint64_t* dbar = &bars[q * C::SUBC < C::HALF ? PB_DA : PB_DB];
    surr_record* mycand = ts.cand + (size_t)wq * CAND_CAP;
    uint32_t ncand = 0, phd = 0, region = 0;
    const float4* w4 = reinterpret_cast<const float4*>(smem + p.off_fin) + q * C::SUBC / 4;
    uint64_t I = p.begin + pair * (2 * TILE_M) + rank * TILE_M + row;
    const bool tw = wq == 0 && lane == 0 && (q == 0 || last);  // trace writers: first and last sub
    uint32_t jt = ~0u;
    for (uint64_t tile = pair; tile < p.num_tiles; tile += npairs) {
      ++jt;
      const bool valid = I < p.end;
    const float accp = ens_prefetch(p, valid, I);
      float part = 0.0f;
      for (uint32_t l = 0; l < p.NL; ++l) {
        const uint32_t dcol = tmem_base + tl + region * H + q * C::SUBC;
        region ^= 1u;
        if (tw && l == 0) trace_ev(p, last ? 2 : 1, jt, 12);
        mbar_wait(dbar, phd);
        phd ^= 1u;
        tc_fence_after();
        if (tw && l < 3) trace_ev(p, last ? 2 : 1, jt, 3 * l);
        if (l + 1 < p.NL) {
          // two K quarters: ReLU + bf16 pack in place, then signal the issuer
#pragma unroll
          for (int j = 0; j < C::QPS; ++j) {
            uint32_t v[C::QC / 32][32];
#pragma unroll
            for (int c = 0; c < C::QC / 32; ++c) tmem_ld32(dcol + j * C::QC + c * 32, v[c]);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < C::QC / 32; ++c) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i)
                pk[i] = relu_pk16<PREC>(__uint_as_float(v[c][2 * i]), __uint_as_float(v[c][2 * i + 1]));
              tmem_st16(dcol + (j * C::QC + c * 32) / 2, pk);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&bars[PB_AQ + C::QPS * q + j], 0);
            if (tw && l < 2) trace_ev(p, last ? 2 : 1, jt, 3 * l + 1 + j);
          }
        } else {
          // final FP32 layer over this sub's columns: w relu(x) = (w/2) x + (w/2) |x|
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int c = 0; c < C::SUBC / 32; c += 2) {
            uint32_t v[2][32];
            tmem_ld32(dcol + c * 32, v[0]);
            tmem_ld32(dcol + (c + 1) * 32, v[1]);
            tmem_wait_ld();
            // region read: the next tile's layer 2 may overwrite it (signalled only
            // where the issuer waits for it: 14-H-1 nets, or subs != 2; an
            // unwaited barrier phase is what compute-sanitizer's synccheck flags)
            if (c + 2 >= C::SUBC / 32 && (p.NL == 1 || C::NSUB != 2)) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_remote(&bars[PB_RF], 0);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const float4 w = w4[((c + u) * 32 + i) / 4];
                const float x0 = __uint_as_float(v[u][i]), x1 = __uint_as_float(v[u][i + 1]);
                const float x2 = __uint_as_float(v[u][i + 2]), x3 = __uint_as_float(v[u][i + 3]);
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
          if (tw) trace_ev(p, last ? 2 : 1, jt, 9);
        }
      }
      // sub 0's partial -> sub 1 through shared memory: barrier 1 = "written"
      // (sub 0 arrives, sub 1 waits), barrier 2 = "consumed" (the reverse), so
      // sub 0 never waits for sub 1's final layer
      if (!last) {
        if (tile != pair) named_bar_sync(2, 128 * C::NSUB);
        red[q * TILE_M + row] = part;
        named_bar_arrive(1, 128 * C::NSUB);
      } else {
        named_bar_sync(1, 128 * C::NSUB);
      }
      if (tw) trace_ev(p, last ? 2 : 1, jt, 10);
      if (last) {
        float t = part;
#pragma unroll
        for (int qq = C::NSUB - 2; qq >= 0; --qq) t += red[qq * TILE_M + row];
        t += p.c_out;
        if (tile + npairs < p.num_tiles) named_bar_arrive(2, 128 * C::NSUB);
        if (!ens_stage(p, valid, I, t, accp)) {
        } else if (mode == MODE_TOPK) {
          topk_offer(ts, mycand, ncand, valid, t, I, p.k, lane);
        } else if (valid && mode != MODE_A0) {
          p.t_dense[I - p.begin] = t;
        }
      }
      if (tw) trace_ev(p, last ? 2 : 1, jt, 11);
      I += dI;
    }
    if (last && mode == MODE_TOPK) topk_post(ts, mycand, ncand, lane);
  }

  // ---- teardown
  tc_fence_before();
  __syncthreads();
  if (mode == MODE_TOPK) {
    topk_drain(ts, p.k, warp, lane);
    __syncthreads();
    const surr_record* L = ts.lists + (size_t)ts.misc[1] * p.k;
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) p.recs[(size_t)blockIdx.x * p.k + i] = L[i];
  }
  cluster_sync();  // the leader's last UMMAs (reading this CTA's TMEM) are complete in both
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
  grid_merge_tail(p, mode, smem);
}

}  // namespace surr
