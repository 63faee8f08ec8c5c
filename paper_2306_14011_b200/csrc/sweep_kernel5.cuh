// K1 for the TF32-family precisions (SURR_PREC_FP32 = 3xTF32 hidden layers,
// SURR_PREC_TF32 = 1xTF32 hidden layers; both with a 3xTF32 first layer),
// nets with at most one hidden->hidden layer, H <= 128.
//
// TMEM per slot: D (H fp32 columns) + A (H columns tf32 hi, + H lo for 3xTF32):
// FP32 = 3H (one slot at H = 128), TF32 = 2H (two slots).  To shorten the
// per-tile dependency chain, each slot's columns are split across NSUB
// warpgroups (TMEM lane quadrant = warp % 4, so a row's columns can be shared
// by several warps but not its lanes): sub q owns columns [q CPS, (q+1) CPS)
// of every epilogue and the final-layer partial over the same columns; the
// partials meet in shared memory and the last sub runs the top-k.  As in the
// BF16 kernel there is no central MMA warp: after the slot's warps pass a
// named barrier, one elected lane of the slot's first warp issues the layer's
// fully unrolled UMMA chain (kind::tf32, A from TMEM) and commits it.
//
// PREC_FP32H: the FP32 path as 3xFP16 (kind::f16 at twice the kind::tf32 rate;
// fp16 hi + fp16 lo carry 22 significant bits, the same as the tf32 split).
// The hidden epilogue packs A = [hi | lo] IN PLACE over the D1 columns it reads
// (32-column chunk c -> 16 hi columns at 32c, 16 lo columns at 32c + 16), the
// last layer accumulates into its own region Y, and the layer-1 operand A0
// (hi and lo tiles) lives in shared memory (SS-form UMMA), so a slot needs
// only 2H columns: two slots at H = 128.
#pragma once
#include "sweep_kernel.cuh"
#include "sweep_kernel3.cuh"  // st_a0_smem

namespace surr {

template <int PREC, int H>
struct Cfg5 {
  static constexpr bool H16 = PREC == PREC_FP32H;  // 3xFP16, A packed in place, A0 in smem
  static constexpr int A_COLS = H16 ? 0 : PREC == PREC_FP32 ? 2 * H : H;
  // FP32: the last layer accumulates into its own region Y = D2, so the next
  // tile's layer-1 UMMA (into D1) overlaps this tile's final layer (reads D2)
  static constexpr bool SEP_Y = PREC == PREC_FP32 || H16;
  static constexpr int SLOT_COLS = H + A_COLS + (SEP_Y ? H : 0);
  static constexpr int Y_COL = H + A_COLS;  // D2 region (SEP_Y)
  static constexpr int NSLOT = 512 / SLOT_COLS >= 2 ? 2 : 1;
  static constexpr int NSUB0 = NSLOT == 2 ? 2 : 4;
  static constexpr int NSUB = (H / 32 < NSUB0) ? H / 32 : NSUB0;  // warpgroups per slot
  static constexpr int CPS = H / NSUB;                            // columns per sub (multiple of 32)
  static constexpr int NEED = NSLOT * SLOT_COLS;
  static constexpr int TMEM_COLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 * NSLOT * NSUB;
  static constexpr int THREE_H = PREC == PREC_FP32 || H16;  // 3 passes in hidden layers
  static constexpr int A0_LO = PREC == PREC_FP32 ? H : K0;
  static_assert(NEED <= 512, "TMEM budget");
};

template <int PREC, int H>
__global__ void __launch_bounds__(Cfg5<PREC, H>::THREADS, 1)
    sweep_kernel5(const __grid_constant__ KParams p, int mode) {
  using C = Cfg5<PREC, H>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);  // [0] load, [4 + s] d ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  // [slot][sub][row] partials (3xFP16: after the shared-memory A0 tiles)
  float* red = reinterpret_cast<float*>(smem + (C::H16 ? p.smem_ones + 4096 : p.smem_a0));
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < C::NSLOT; ++s) mbar_init(&bars[4 + s], 1);
      if (C::H16)  // 3xFP16: separate "L2 done" barriers (the next L1 is issued without a slot barrier)
        for (int s = 0; s < C::NSLOT; ++s) mbar_init(&bars[6 + s], 1);
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint32_t total = p.w_bytes + (mode == MODE_PREDICT ? 0u : p.lut_bytes);
      mbar_arrive_expect_tx(&bars[0], total);
      for (uint32_t off = 0; off < p.w_bytes; off += 32768u)
        bulk_g2s(smem + off, (const uint8_t*)p.w_gmem + off, min(32768u, p.w_bytes - off), &bars[0]);
      if (mode != MODE_PREDICT && p.lut_bytes) bulk_g2s(smem + p.smem_lut, p.lut_gmem, p.lut_bytes, &bars[0]);
    }
    __syncwarp();
    tmem_alloc<C::TMEM_COLS>(tmem_slot);
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // ---- roles: warpgroup wg = s * NSUB + q
  const uint32_t wg = warp >> 2;
  const uint32_t s = wg / C::NSUB;
  const uint32_t q = wg % C::NSUB;
  const bool first = q == 0, last = q == C::NSUB - 1;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t tl = (wq * 32u) << 16;
  const uint32_t dslot = tmem_base + s * C::SLOT_COLS;  // lane-0 view (UMMA operands)
  const uint32_t dcol = dslot + tl + q * C::CPS;         // this warp's D columns
  const uint32_t acol = dslot + tl + (C::H16 ? 0 : H);   // this warp's A region
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)(s * 4 + wq) * CAND_CAP;
  uint32_t ncand = 0;
  const uint32_t bar_id = 1 + s;
  const bool issuer = first && wq == 0;
  const uint32_t sb = smem_u32(smem);
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint64_t d_b1lo = make_bdesc(sb + p.off_b1lo, p.sbo_b1);
  const uint64_t d_b2 = make_bdesc(sb + p.off_bh, p.sbo_bh);
  const uint64_t d_b2lo = make_bdesc(sb + p.off_bh + p.lo_delta_h, p.sbo_bh);
  const uint32_t idesc = p.idesc;
  uint8_t* a0h_tile = smem + p.smem_a0 + s * 2 * 4096;  // 3xFP16: A0 hi / lo tiles of this slot
  uint8_t* a0l_tile = a0h_tile + 4096;
  const uint64_t d_a0h = make_bdesc(sb + p.smem_a0 + s * 2 * 4096, 256);
  const uint64_t d_a0l = make_bdesc(sb + p.smem_a0 + s * 2 * 4096 + 4096, 256);

  // one elected thread of the issuer warp: the layer's UMMA chain + commit
  auto mma_chain = [&](int layer) {
        const uint32_t a = dslot + H;
        if (C::H16 && layer == 0) {
          umma_f16_ss(dslot, d_a0h, d_b1, idesc, 0u);
          umma_f16_ss(dslot, d_a0l, d_b1, idesc, 1u);
          umma_f16_ss(dslot, d_a0h, d_b1lo, idesc, 1u);
        } else if (C::H16) {
          // layer l reads A (packed in place) from region (l - 1) & 1 and writes region
          // l & 1 (D1 = region 0, Y = region 1): ping-pong for nets with > 1 hidden->hidden layer
          const uint32_t d2 = dslot + (layer & 1) * H;
          const uint32_t asrc = dslot + ((layer - 1) & 1) * H;
          const uint64_t bh = d_b2 + (uint64_t)((((uint32_t)layer - 1) * p.stride_bh) >> 4);
          const uint64_t bl = d_b2lo + (uint64_t)((((uint32_t)layer - 1) * p.stride_bh) >> 4);
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk) {
            const uint32_t ah = asrc + 32 * (kk >> 1) + 8 * (kk & 1);  // hi; lo at + 16
            umma_f16_ts(d2, ah, bh + kk * 16, idesc, kk > 0);
            umma_f16_ts(d2, ah + 16, bh + kk * 16, idesc, 1u);
            umma_f16_ts(d2, ah, bl + kk * 16, idesc, 1u);
          }
        } else if (layer == 0) {
#pragma unroll
          for (int kk = 0; kk < K0 / 8; ++kk) {
            umma_tf32_ts(dslot, a + kk * 8, d_b1 + kk * 16, idesc, kk > 0);
            umma_tf32_ts(dslot, a + kk * 8, d_b1lo + kk * 16, idesc, 1u);
            umma_tf32_ts(dslot, a + C::A0_LO + kk * 8, d_b1 + kk * 16, idesc, 1u);
          }
        } else {
          const uint32_t d2 = dslot + (C::SEP_Y ? C::Y_COL : 0);
#pragma unroll
          for (int kk = 0; kk < H / 8; ++kk) {
            umma_tf32_ts(d2, a + kk * 8, d_b2 + kk * 16, idesc, kk > 0);
            if (C::THREE_H) {
              umma_tf32_ts(d2, a + kk * 8, d_b2lo + kk * 16, idesc, 1u);
              umma_tf32_ts(d2, a + H + kk * 8, d_b2 + kk * 16, idesc, 1u);
            }
          }
        }
        umma_commit(&bars[(C::H16 && layer == 1 && p.NL == 2) ? 6 + s : 4 + s]);
  };
  auto issue = [&](int layer) {
    tc_fence_before();
    named_bar_sync(bar_id, 128 * C::NSUB);
    if (issuer) {
      tc_fence_after();
      if (elect_one()) mma_chain(layer);
      __syncwarp();
    }
  };

  uint64_t tile = (uint64_t)blockIdx.x * C::NSLOT + s;
  uint64_t I = p.begin + tile * TILE_M + row;
  const uint64_t dI = (uint64_t)p.dTiles * TILE_M;
  uint32_t D[MAXG];
  if (first && mode != MODE_PREDICT) init_digits(p.R, I, D);
  uint32_t phd = 0, phd2 = 0;
  mbar_wait(&bars[0], 0);

  A0Regs a0;
  auto put_a0 = [&]() {  // sub 0 stores the layer-1 operand (tf32 hi / lo slots, or fp16 tiles)
    if (C::H16) {
      st_a0_smem(a0h_tile, row, a0.hi);
      st_a0_smem(a0l_tile, row, a0.lo);
      fence_proxy_async_smem();
    } else {
      tmem_st16(acol, a0.hi);
      tmem_st16(acol + C::A0_LO, a0.lo);
      tmem_wait_st();
    }
  };
  // separate Y region only with a hidden->hidden layer (14-H-1 nets: the final
  // layer reads D1, and the next L1 waits for those reads at the slot barrier)
  const bool sep = C::SEP_Y && p.NL == 2;
  if (first && tile < p.num_tiles) {
    if (mode == MODE_PREDICT) make_a0_predict<PREC>(p, I < p.end ? I : p.begin, a0);
    else make_a0_sweep<PREC>(p, slut, D, a0);
    put_a0();
  }
  if (tile < p.num_tiles) issue(0);
  uint32_t jr = 0;
  for (; tile < p.num_tiles; tile += p.dTiles, ++jr) {
    const bool tr = q == 0 && wq == 0 && lane == 0;
    if (tr) trace_ev(p, s, jr, 0);
    const bool valid = I < p.end;
    const float accp = ens_prefetch(p, valid, I);
    const uint64_t In = I + dI;
    const bool has_next = tile + p.dTiles < p.num_tiles;
    float part = 0.0f;
    for (uint32_t l = 0; l < p.NL; ++l) {
      if (C::H16 && l == 1 && p.NL == 2) {
        mbar_wait(&bars[6 + s], phd2);
        phd2 ^= 1u;
      } else {
        mbar_wait(&bars[4 + s], phd);
        phd ^= 1u;
      }
      tc_fence_after();
      if (tr) trace_ev(p, s, jr, 1 + 2 * l);
      if (l + 1 < p.NL) {
        // a5: hidden epilogue over this sub's columns -> A (tf32 hi [, lo])
#pragma unroll
        for (int c = 0; C::H16 && c < C::CPS / 32; ++c) {
          // in place: chunk c (32 fp32 columns, read first) -> 16 hi + 16 lo fp16x2 columns
          // of region l & 1; layers l >= 1 add their bias here (layer 1's rides in A0)
          const uint32_t rcol = dcol + (l & 1u) * H;
          uint32_t v[32];
          tmem_ld32(rcol + c * 32, v);
          tmem_wait_ld();
          uint32_t hv[16], lv[16];
          const int col0 = (int)(q * C::CPS) + c * 32;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float y0 = __uint_as_float(v[2 * j]), y1 = __uint_as_float(v[2 * j + 1]);
            if (l >= 1) {
              y0 += p.hbias[(l - 1) & 1][col0 + 2 * j];
              y1 += p.hbias[(l - 1) & 1][col0 + 2 * j + 1];
            }
            const float x0 = fmaxf(y0, 0.0f), x1 = fmaxf(y1, 0.0f);
            hv[j] = f16x2(x0, x1);
            float h0, h1;
            f16x2_to_f32(hv[j], h0, h1);
            lv[j] = f16x2(x0 - h0, x1 - h1);  // x - hi is exact in fp32; one rounding to fp16
          }
          tmem_st16(rcol + c * 32, hv);
          tmem_st16(rcol + c * 32 + 16, lv);
        }
#pragma unroll
        for (int c = 0; !C::H16 && c < C::CPS / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(dcol + c * 32, v);
          tmem_wait_ld();
          uint32_t hv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = fmaxf(__uint_as_float(v[j]), 0.0f);  // layer-1 bias rides in A0's ones slot
            hv[j] = to_tf32(x);
            if (C::THREE_H) v[j] = __float_as_uint(x - __uint_as_float(hv[j]));  // exact; truncated by the UMMA
          }
          tmem_st32(acol + q * C::CPS + c * 32, hv);
          if (C::THREE_H) tmem_st32(acol + H + q * C::CPS + c * 32, v);
        }
        tmem_wait_st();
        if (tr) trace_ev(p, s, jr, 2);
        issue((int)l + 1);  // the next layer (nets deeper than two layers: l + 1 > 1)
        if (C::H16 && sep && first && has_next) {
          // 3xFP16: L1 of this tile is done, so the next tile's A0 tiles (shared
          // memory) can be written now; sub 0's warps sync among themselves and
          // the issuer starts the next L1 the moment L2 completes
          if (mode == MODE_PREDICT) {
            make_a0_predict<PREC>(p, In < p.end ? In : p.begin, a0);
          } else {
            odometer_step(p.R, p.dD, D);
            make_a0_sweep<PREC>(p, slut, D, a0);
          }
          put_a0();
          named_bar_sync(3 + s, 128);
        } else if (sep && first && has_next) {  // next tile's digits / row while L2 runs
          if (mode == MODE_PREDICT) make_a0_predict<PREC>(p, In < p.end ? In : p.begin, a0);
          else odometer_step(p.R, p.dD, D);
        }
      } else {
        // a7: final-layer partial over this sub's columns (relu(x + b) = max(x, -b) + b)
        if (C::H16 && sep && has_next) {
          // L2 done (A free): the next tile's L1 into D1 while Y is read; its A0
          // tiles were stored (and synced within sub 0) while L2 ran.  The L1 and
          // L2 completions use separate mbarriers, so no slot barrier is needed
          if (issuer) {
            if (elect_one()) mma_chain(0);
            __syncwarp();
          }
        } else if (sep && has_next) {
          // D2 ready => L2 no longer reads A: store the next A0 there and start
          // the next tile's layer 1 (into D1) before reading D2
          if (first) {
            if (mode != MODE_PREDICT) make_a0_sweep<PREC>(p, slut, D, a0);
            put_a0();
          }
          issue(0);
        }
        // the last layer's region: Y for the two-layer split, else by layer parity (3xFP16)
        const uint32_t fcol = dcol + (C::H16 ? ((p.NL - 1) & 1u) * H : (sep ? C::Y_COL : 0));
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int c = 0; c < C::CPS / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(fcol + c * 32, v);
          tmem_wait_ld();
          // w and -b of this sub's columns: broadcast 16-byte shared-memory loads
          // (the column offset depends on the warpgroup, so no constant-bank operands)
          const float4* w4 = reinterpret_cast<const float4*>(smem + p.off_fin) + (q * C::CPS + c * 32) / 4;
          const float4* nb4 = w4 + H / 4;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 w = w4[j / 4], nb = nb4[j / 4];
            const float x0 = fmaxf(__uint_as_float(v[j]), nb.x), x1 = fmaxf(__uint_as_float(v[j + 1]), nb.y);
            const float x2 = fmaxf(__uint_as_float(v[j + 2]), nb.z), x3 = fmaxf(__uint_as_float(v[j + 3]), nb.w);
            acc[(j >> 2) & 1] = ffma2(pack2(w.x, w.y), pack2(x0, x1), acc[(j >> 2) & 1]);
            acc[2 + ((j >> 2) & 1)] = ffma2(pack2(w.z, w.w), pack2(x2, x3), acc[2 + ((j >> 2) & 1)]);
          }
        }
        float a8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
        part = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
      }
    }
    // next tile's A0 (sub 0) and the next layer-1 UMMA as soon as D is free
    if (!sep && first && has_next) {
      if (mode == MODE_PREDICT) {
        make_a0_predict<PREC>(p, In < p.end ? In : p.begin, a0);
      } else {
        odometer_step(p.R, p.dD, D);
        make_a0_sweep<PREC>(p, slut, D, a0);
      }
      put_a0();
    }
    if (tr) trace_ev(p, s, jr, 5);
    if (C::NSUB > 1 && !last) red[(s * C::NSUB + q) * TILE_M + row] = part;
    if (!sep && has_next) issue(0);  // includes the slot barrier: partials are visible after it
    else named_bar_sync(bar_id, 128 * C::NSUB);
    if (tr) trace_ev(p, s, jr, 6);
    if (last) {
      float t = 0.0f;
#pragma unroll
      for (int qq = 0; qq + 1 < C::NSUB; ++qq) t += red[(s * C::NSUB + qq) * TILE_M + row];
      t = t + part + p.c_out;
      if (!ens_stage(p, valid, I, t, accp)) {
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
  if (last && mode == MODE_TOPK) topk_post(ts, mycand, ncand, lane);

  // ---- teardown
  tc_fence_before();
  __syncthreads();
  if (mode == MODE_TOPK) {
    topk_drain(ts, p.k, warp, lane);
    __syncthreads();
    const surr_record* L = ts.lists + (size_t)ts.misc[1] * p.k;
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) p.recs[(size_t)blockIdx.x * p.k + i] = L[i];
  }
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  grid_merge_tail(p, mode, smem);
}

}  // namespace surr
