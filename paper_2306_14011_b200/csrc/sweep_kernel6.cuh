// K1 for the FP32 path as 3xFP16 with THREE tiles in flight per SM (nets with
// one hidden->hidden layer, H <= 128: every BASELINE net on the FP32 path).
//
// The 2-slot kernel (sweep_kernel5<PREC_FP32H>) keeps each slot's last layer
// in its own H-column region Y, so TMEM (2 x (H + H)) holds two tiles and the
// tensor pipe idles whenever both slots are in their CUDA-core phases (ncu:
// ~61 % tensor-pipe activity).  Here the three slots own only their D1/A
// regions (H columns each: the layer-1 accumulator, then A = [hi | lo] packed
// in place) and SHARE one last-layer region Y, split in two N-halves Y0, Y1:
//
//   slot s, tile j:  L1 -> epi1 (in place) -> [wait Y0 free] L2a -> Y0
//                                          -> [wait Y1 free] L2b -> Y1
//                    read Y0 -> release Y0 -> FP32 partial a
//                    read Y1 -> release Y1 -> (next L1) -> FP32 partial b -> top-k
//
// The halves make the hand-over overlap: while slot s's L2b runs, slot s
// reads and releases Y0, so the next slot's L2a starts right after L2b; while
// that runs, slot s releases Y1.  The users of Y0 / Y1 go round robin
// (slot 0, 1, 2, 0, ...): "Y_h released by slot s" is one mbarrier per (half,
// slot) that completes once per tile, and the issuer of slot s waits for its
// predecessor's release of the same round (slot 0: the previous round of
// slot 2).  A waiter is never more than one phase behind (the next release of
// that slot needs this slot's own release first), so parity waits are exact.
// Every slot runs the same number of rounds (the CTA's slot-0 count); a slot
// whose tile is past the end runs a masked dummy tile so the round robin
// never stalls.  One warpgroup per slot (384 threads, no register cap issue).
#pragma once
#include "sweep_kernel.cuh"
#include "sweep_kernel3.cuh"  // st_a0_smem, topk_offer

namespace surr {

template <int H>
struct Cfg6 {
  static constexpr int NSLOT = 3;
  static constexpr int THREADS = 128 * NSLOT;
  static constexpr int Y_COL = NSLOT * H;  // shared last-layer region [Y_COL, Y_COL + H)
  static constexpr int NEED = NSLOT * H + H;
  static constexpr int TMEM_COLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static_assert(NEED <= 512, "TMEM budget");
  static_assert(H % 32 == 0 && H <= 128, "H");
};

// mbarrier indices (the misc area holds 64 of them; 8 = TMEM slot word, 16.. = top-k scalars)
enum { K6_LOAD = 0, K6_L1 = 32, K6_L2A = 35, K6_L2B = 38, K6_Y0F = 41, K6_Y1F = 44 };

template <int H>
__global__ void __launch_bounds__(Cfg6<H>::THREADS, 1) sweep_kernel6(const __grid_constant__ KParams p, int mode) {
  using C = Cfg6<H>;
  constexpr int HH = H / 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[K6_LOAD], 1);
      for (int s = 0; s < C::NSLOT; ++s) {
        mbar_init(&bars[K6_L1 + s], 1);
        mbar_init(&bars[K6_L2A + s], 1);
        mbar_init(&bars[K6_L2B + s], 1);
        mbar_init(&bars[K6_Y0F + s], 4);  // the slot's four warps release
        mbar_init(&bars[K6_Y1F + s], 4);
      }
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint32_t total = p.w_bytes + (mode == MODE_PREDICT ? 0u : p.lut_bytes);
      mbar_arrive_expect_tx(&bars[K6_LOAD], total);
      for (uint32_t off = 0; off < p.w_bytes; off += 32768u)
        bulk_g2s(smem + off, (const uint8_t*)p.w_gmem + off, min(32768u, p.w_bytes - off), &bars[K6_LOAD]);
      if (mode != MODE_PREDICT && p.lut_bytes) bulk_g2s(smem + p.smem_lut, p.lut_gmem, p.lut_bytes, &bars[K6_LOAD]);
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

  // ---- slot roles
  const uint32_t s = warp >> 2;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t tl = (wq * 32u) << 16;
  const uint32_t dslot = tmem_base + s * H;        // lane-0 view: D1 / A of this slot
  const uint32_t dcol = dslot + tl;                // this warp's lanes
  const uint32_t ycol = tmem_base + tl + C::Y_COL;  // this warp's lanes of Y
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)warp * CAND_CAP;
  uint32_t ncand = 0;
  const uint32_t bar_id = 1 + s;
  const bool issuer = wq == 0;
  const uint32_t sb = smem_u32(smem);
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint64_t d_b1lo = make_bdesc(sb + p.off_b1lo, p.sbo_b1);
  const uint64_t d_b2a = make_bdesc(sb + p.off_bh, p.sbo_bh);
  const uint64_t d_b2alo = make_bdesc(sb + p.off_bh + p.lo_delta_h, p.sbo_bh);
  const uint64_t d_b2b = make_bdesc(sb + p.off_bh + (uint32_t)(HH / 8) * p.sbo_bh, p.sbo_bh);
  const uint64_t d_b2blo = make_bdesc(sb + p.off_bh + (uint32_t)(HH / 8) * p.sbo_bh + p.lo_delta_h, p.sbo_bh);
  const uint32_t idesc = p.idesc;
  const uint32_t idesc_half = (idesc & ~(0x3Fu << 17)) | (((uint32_t)HH >> 3) << 17);
  uint8_t* a0h_tile = smem + p.smem_a0 + s * 2 * 4096;
  uint8_t* a0l_tile = a0h_tile + 4096;
  const uint64_t d_a0h = make_bdesc(sb + p.smem_a0 + s * 2 * 4096, 256);
  const uint64_t d_a0l = make_bdesc(sb + p.smem_a0 + s * 2 * 4096 + 4096, 256);
  const uint32_t prev = (s + C::NSLOT - 1) % C::NSLOT;  // the slot that used Y before us in a round

  auto l1_chain = [&]() {  // one elected thread
    umma_f16_ss(dslot, d_a0h, d_b1, idesc, 0u);
    umma_f16_ss(dslot, d_a0l, d_b1, idesc, 1u);
    umma_f16_ss(dslot, d_a0h, d_b1lo, idesc, 1u);
    umma_commit(&bars[K6_L1 + s]);
  };
  auto l2_chain = [&](int hh) {  // one elected thread: output neurons [hh H/2, (hh+1) H/2) -> Y_hh
    const uint32_t d2 = tmem_base + C::Y_COL + hh * HH;
    const uint64_t bh = hh ? d_b2b : d_b2a, bl = hh ? d_b2blo : d_b2alo;
#pragma unroll
    for (int kk = 0; kk < H / 16; ++kk) {
      const uint32_t ah = dslot + 32 * (kk >> 1) + 8 * (kk & 1);  // hi; lo at + 16
      umma_f16_ts(d2, ah, bh + kk * 16, idesc_half, kk > 0);
      umma_f16_ts(d2, ah + 16, bh + kk * 16, idesc_half, 1u);
      umma_f16_ts(d2, ah, bl + kk * 16, idesc_half, 1u);
    }
    umma_commit(&bars[(hh ? K6_L2B : K6_L2A) + s]);
  };
  auto wait_bar = [&](uint32_t idx, uint32_t par) {
    mbar_wait(&bars[idx], par);
    tc_fence_after();
  };
  // FP32 final-layer partial over HH columns of Y half hh (loaded by the caller):
  // relu(x + b) = max(x, -b) + b with w, -b broadcast from shared memory
  auto fin_half = [&](const uint32_t (&v)[HH], int hh) -> float {
    const float4* w4 = reinterpret_cast<const float4*>(smem + p.off_fin) + hh * HH / 4;
    const float4* nb4 = w4 + H / 4;
    uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int j = 0; j < HH; j += 4) {
      const float4 w = w4[j / 4], nb = nb4[j / 4];
      const float x0 = fmaxf(__uint_as_float(v[j]), nb.x), x1 = fmaxf(__uint_as_float(v[j + 1]), nb.y);
      const float x2 = fmaxf(__uint_as_float(v[j + 2]), nb.z), x3 = fmaxf(__uint_as_float(v[j + 3]), nb.w);
      acc[(j >> 2) & 1] = ffma2(pack2(w.x, w.y), pack2(x0, x1), acc[(j >> 2) & 1]);
      acc[2 + ((j >> 2) & 1)] = ffma2(pack2(w.z, w.w), pack2(x2, x3), acc[2 + ((j >> 2) & 1)]);
    }
    float a8[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
    return ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
  };
  auto load_half = [&](uint32_t (&v)[HH], int hh) {
    if (HH >= 32) {
#pragma unroll
      for (int c = 0; c < HH / 32; ++c) tmem_ld32(ycol + hh * HH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[c * 32]));
    } else {
      tmem_ld16(ycol + hh * HH, v);
    }
    tmem_wait_ld();
  };

  // ---- tile schedule: every slot runs the CTA's slot-0 round count
  const uint64_t t0 = (uint64_t)blockIdx.x * C::NSLOT;
  const uint32_t rounds = t0 < p.num_tiles ? (uint32_t)((p.num_tiles - t0 - 1) / p.dTiles + 1) : 0u;
  uint64_t tile = t0 + s;
  uint64_t I = p.begin + tile * TILE_M + row;
  const uint64_t dI = (uint64_t)p.dTiles * TILE_M;
  uint32_t D[MAXG];
  if (mode != MODE_PREDICT) init_digits(p.R, I, D);
  mbar_wait(&bars[K6_LOAD], 0);

  A0Regs a0;
  auto put_a0 = [&]() {
    st_a0_smem(a0h_tile, row, a0.hi);
    st_a0_smem(a0l_tile, row, a0.lo);
    fence_proxy_async_smem();
  };
  auto make_a0 = [&](uint64_t Ir) {
    if (mode == MODE_PREDICT) make_a0_predict<PREC_FP32H>(p, Ir < p.end ? Ir : p.begin, a0);
    else make_a0_sweep<PREC_FP32H>(p, slut, D, a0);
    if (mode != MODE_PREDICT) a0_dump<true>(p, mode, a0, Ir);
  };
  if (rounds) {
    make_a0(I);
    put_a0();
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (issuer) {
      tc_fence_after();
      if (elect_one()) l1_chain();
      __syncwarp();
    }
  }
  for (uint32_t j = 0; j < rounds; ++j, tile += p.dTiles) {
    const uint32_t par = j & 1u;
    const bool valid = tile < p.num_tiles && I < p.end;
    const float accp = ens_prefetch(p, valid, I);
    const uint64_t In = I + dI;
    const bool has_next = j + 1 < rounds;

    wait_bar(K6_L1 + s, par);  // L1 done: D1 holds the layer-1 pre-activations, A0 tiles are free
    // a5 in place: chunk c (32 fp32 columns, read first) -> 16 hi + 16 lo fp16x2 columns
#pragma unroll
    for (int c = 0; c < H / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(dcol + c * 32, v);
      tmem_wait_ld();
      uint32_t hv[16], lv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float x0 = fmaxf(__uint_as_float(v[2 * q]), 0.0f), x1 = fmaxf(__uint_as_float(v[2 * q + 1]), 0.0f);
        hv[q] = f16x2(x0, x1);
        float h0, h1;
        f16x2_to_f32(hv[q], h0, h1);
        lv[q] = f16x2(x0 - h0, x1 - h1);  // x - hi is exact in fp32; one rounding to fp16
      }
      tmem_st16(dcol + c * 32, hv);
      tmem_st16(dcol + c * 32 + 16, lv);
    }
    tmem_wait_st();
    if (has_next) {  // the next tile's A0 (its L1 is issued the moment L2b completes)
      if (mode != MODE_PREDICT) odometer_step(p.R, p.dD, D);
      make_a0(In);
      put_a0();
    }
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (issuer) {
      tc_fence_after();
      // Y round robin: use (j, s) follows (j, s - 1), or (j - 1, 2) for slot 0
      const bool first_use = (j == 0 && s == 0);
      const uint32_t ppar = (s == 0 ? j - 1 : j) & 1u;
      if (!first_use) mbar_wait(&bars[K6_Y0F + prev], ppar);
      tc_fence_after();
      if (elect_one()) l2_chain(0);
      __syncwarp();
      if (!first_use) mbar_wait(&bars[K6_Y1F + prev], ppar);
      tc_fence_after();
      if (elect_one()) l2_chain(1);
      __syncwarp();
    }
    float part;
    {
      uint32_t v[HH];
      wait_bar(K6_L2A + s, par);
      load_half(v, 0);
      tc_fence_before();
      __syncwarp();
      // Y0 read: the next user may overwrite it (the very last use has no next user)
      const bool release = !(j + 1 == rounds && s == C::NSLOT - 1);
      if (lane == 0 && release) mbar_arrive(&bars[K6_Y0F + s]);
      part = fin_half(v, 0);
    }
    {
      uint32_t v[HH];
      wait_bar(K6_L2B + s, par);
      load_half(v, 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && !(j + 1 == rounds && s == C::NSLOT - 1)) mbar_arrive(&bars[K6_Y1F + s]);
      if (issuer && has_next) {  // L2b done: A (D1) is free; A0 was stored before the slot barrier
        if (elect_one()) l1_chain();
        __syncwarp();
      }
      part += fin_half(v, 1);
    }
    float t = part + p.c_out;
    if (!ens_stage(p, valid, I, t, accp)) {
    } else if (mode == MODE_TOPK) {
      topk_offer(ts, mycand, ncand, valid, t, I, p.k, lane);
    } else if (valid && mode != MODE_A0) {
      p.t_dense[I - p.begin] = t;
    }
    I = In;
  }
  if (mode == MODE_TOPK) topk_post(ts, mycand, ncand, lane);

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
