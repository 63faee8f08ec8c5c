// K1, 16-bit variant (FP16 with PREC = PREC_FP16, or BF16) with NS = 4 128-row
// tiles in flight per SM (nets with at most one hidden->hidden layer: 14-H-1
// and 14-H-H-1, H <= 128).
//
// TMEM per slot is just the H-column accumulator region D:
//   L1   : D[0, H)      = A0 x [W1; b1]                               (N = H)
//   epi1 : ReLU + 16-bit pack of D[0, H) written IN PLACE to D[0, H/2): a
//          thread reads chunk c (32 columns) before writing packed chunk c to
//          columns 16c .. 16c+15, which it has already read, so A1 needs no columns
//   L2a  : D[H/2, H)    = A1 x [W2; b2] (output neurons 0 .. H/2-1)     (N = H/2)
//   fin-a: FP32 partial dot product over those neurons, then D[H/2, H) is free
//   L2b  : D[H/2, H)    = A1 x [W2; b2] (output neurons H/2 .. H-1)
//   fin-b: rest of the dot product, de-standardise, top-k
// With NS = 4 the layer-1 operand A0 and the bias ones block live in shared
// memory (SS-form UMMA for those two small steps), so 4 slots x H = all 512
// columns at H = 128.  The next tile's A0 is decoded and stored while L2b runs.
// The ENS instantiation (ensemble members >= 1) stages the member's fp32
// accumulator slice of the tile into shared memory with a bulk copy issued
// with the tile's L1.
//
// There is no central MMA warp: each slot's warpgroup issues its own UMMAs.
// After the four warps finish writing (tcgen05.st) or reading (tcgen05.ld)
// the slot's TMEM they meet at a 128-thread named barrier, then one elected
// lane of the slot's first warp issues the phase's UMMA chain and commits it
// to the slot's "D ready" mbarrier, which all four warps wait on.  A measured
// timeline (scripts/trace_timeline.py) showed a single issuer thread
// serialising ~150-400 cycles of wait / fence / issue per phase across slots.
#pragma once
#include "sweep_kernel.cuh"

namespace surr {

template <int H, int NS = 3>
struct Cfg3 {
  static constexpr int NSLOT = NS;
  // NS = 4: the layer-1 operand A0 and the bias ones block live in shared
  // memory (SS-form UMMA for those two small steps) so that the four H-column
  // accumulator regions alone fill TMEM
  static constexpr bool A0_SMEM = NS * H + NS * 8 + 8 > 512;
  static constexpr int A0_COL = NSLOT * H;           // + 8 * slot (TMEM variant)
  static constexpr int ONES_COL = NSLOT * H + 8 * NSLOT;
  static constexpr int NEED = A0_SMEM ? NSLOT * H : ONES_COL + 8;
  static constexpr int TMEM_COLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 * NSLOT;
  static constexpr int A0_TILE_BYTES = 128 * 16 * 2;  // 128 rows x K 16 bf16, K-major core matrices
  static_assert(NEED <= 512, "TMEM budget");
  static_assert(H % 32 == 0 && H <= 128, "H");
};

// A0 row -> shared-memory operand tile (K-major, no swizzle: 8-row x 16-byte
// core matrices, K halves 128 B apart (LBO), 8-row groups 256 B apart (SBO))
__device__ __forceinline__ void st_a0_smem(uint8_t* tile, uint32_t row, const uint32_t* cols8) {
  uint8_t* base = tile + (row >> 3) * 256 + (row & 7) * 16;
  *reinterpret_cast<uint4*>(base) = make_uint4(cols8[0], cols8[1], cols8[2], cols8[3]);
  *reinterpret_cast<uint4*>(base + 128) = make_uint4(cols8[4], cols8[5], cols8[6], cols8[7]);
}

// a8 for one row: ballot filter, per-warp candidate buffer, merge when full
__device__ __forceinline__ void topk_offer(TopkShared& ts, surr_record* mycand, uint32_t& ncand, bool valid, float t,
                                           uint64_t I, uint32_t k, uint32_t lane) {
  const uint32_t key = f2key(t);
  // conservative filter on the key alone (a stale read only admits extra
  // candidates; the merge keeps the exact (key, idx) top-k)
  const bool pass = valid && key <= ts.misc[2];
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, pass);
  if (m) {
    const uint32_t n = __popc(m);
    if (ncand + n > CAND_CAP) {
      lock_acquire(ts, lane);
      warp_merge(ts, mycand, ncand, k, lane);
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
}

// acc += w relu(x) for a column pair, as (w/2) x + (w/2) |x|: two FFMA2, |x| is
// a free operand modifier (fin_w holds y_scale * w / 2)
__device__ __forceinline__ void relu_dot2(const KParams& p, uint32_t v0, uint32_t v1, int n, uint64_t (&acc)[4], int j) {
  const uint64_t w2 = pack2(p.fin_w[n], p.fin_w[n + 1]);
  const float x0 = __uint_as_float(v0), x1 = __uint_as_float(v1);
  acc[(j >> 1) & 1] = ffma2(w2, pack2(x0, x1), acc[(j >> 1) & 1]);
  acc[2 + ((j >> 1) & 1)] = ffma2(w2, pack2(fabsf(x0), fabsf(x1)), acc[2 + ((j >> 1) & 1)]);
}

// FP32 partial of the final layer over NC columns starting at TMEM column
// `col`, output neurons starting at n0 (bias already in D: ReLU threshold 0)
template <int NC>
__device__ __forceinline__ float final_partial(const KParams& p, uint32_t col, int n0) {
  uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
  if (NC == 16) {
    uint32_t v[16];
    tmem_ld16(col, v);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; j += 2) relu_dot2(p, v[j], v[j + 1], n0 + j, acc, j);
  }
#pragma unroll
  for (int c = 0; c < NC / 32; c += 2) {
    uint32_t v[2][32];
    tmem_ld32(col + c * 32, v[0]);
    if (NC / 32 > 1) tmem_ld32(col + (c + 1) * 32, v[1]);
    tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && NC / 32 == 1) break;
      const int base = n0 + (c + u) * 32;
#pragma unroll
      for (int j = 0; j < 32; j += 2) relu_dot2(p, v[u][j], v[u][j + 1], base + j, acc, j);
    }
  }
  float a8[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
  return ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
}

// split form of final_partial for NC <= 64: load (then the caller may release
// the TMEM columns and issue the next UMMA) and compute from registers
template <int NC>
__device__ __forceinline__ void final_load(uint32_t col, uint32_t (&v)[64]) {
  if (NC == 16) {
    tmem_ld16(col, v);
  } else {
    tmem_ld32(col, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
    if (NC == 64) tmem_ld32(col + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
  }
  tmem_wait_ld();
}
template <int NC>
__device__ __forceinline__ float final_compute(const KParams& p, const uint32_t (&v)[64], int n0) {
  uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int j = 0; j < NC; j += 2) relu_dot2(p, v[j], v[j + 1], n0 + j, acc, j);
  float a8[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
  return ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
}

// ENS: the ensemble-member instantiation (accumulator staging compiled in; the
// single-net kernels carry none of it: it cost 4 % on cfg2 in a same-box A/B)
template <int H, int SPG, int NS, int PREC = PREC_BF16, bool ENS = false>
__global__ void __launch_bounds__(Cfg3<H, NS>::THREADS, 1)
    sweep_kernel3(const __grid_constant__ KParams p, int mode) {
  // SPG = parameter slots per decoder group: 4 (two A0 columns per 8-byte table
  // entry, 4 odometer digits) when the table fits, else 2 (8 digits)
  // SPG = 0: the explicit-batch (predict) instantiation, whose rows come from
  // HBM; sweep instantiations carry no predict code (register budget)
  constexpr bool PRED = SPG == 0;
  constexpr int NG = PRED ? 1 : K0 / SPG;
  using C = Cfg3<H, NS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);  // [0] load, [4..6] d ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < C::NSLOT; ++s) mbar_init(&bars[4 + s], 1);
      if (PRED)
        for (int s = 0; s < C::NSLOT; ++s) mbar_init(&bars[9 + s], 1);  // row staging (tmem_slot is at +64)
      for (int s = 0; s < 2 * C::NSLOT; ++s) mbar_init(&bars[32 + s], 1);  // ensemble accumulator staging
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
  if (warp < 4) {
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = one16<PREC>();  // 1.0 in K slot 0
    if (C::A0_SMEM) {
      st_a0_smem(smem + p.smem_ones, warp * 32u + lane, ones);
      fence_proxy_async_smem();
    } else {
      tmem_st8(tmem_base + ((warp * 32u) << 16) + C::ONES_COL, ones);
      tmem_wait_st();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ================= slot warpgroups (self-issuing) =================
  const uint32_t s = warp >> 2;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t tl = (wq * 32u) << 16;
  const uint32_t dslot = tmem_base + s * H;                 // lane 0 view (UMMA operands)
  const uint32_t dcol = dslot + tl;                          // this warp's lanes
  const uint32_t a0col = tmem_base + tl + C::A0_COL + 8 * s;
  uint8_t* a0tile = smem + p.smem_a0 + s * C::A0_TILE_BYTES;
  // A0 of this warp's row -> TMEM (st only; caller waits) or shared memory (+ proxy fence)
  auto put_a0 = [&](const A0Regs& a) {
    if (C::A0_SMEM) {
      st_a0_smem(a0tile, row, a.hi);
      fence_proxy_async_smem();
    } else {
      tmem_st8(a0col, a.hi);
    }
  };
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)warp * CAND_CAP;
  uint32_t ncand = 0;
  const uint32_t bar_id = 1 + s;
  const bool issuer = wq == 0;
  // UMMA operands (warp-uniform)
  const uint32_t sb = smem_u32(smem);
  const uint32_t ones = tmem_base + C::ONES_COL;
  const uint64_t d_ones = make_bdesc(sb + p.smem_ones, 256);
  const uint64_t d_a0 = make_bdesc(sb + p.smem_a0 + s * C::A0_TILE_BYTES, 256);
  const uint32_t idesc_full = p.idesc;
  const uint32_t idesc_half = (p.idesc & ~(0x3Fu << 17)) | (((uint32_t)(H / 2) >> 3) << 17);
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint64_t d_b2a = make_bdesc(sb + p.off_bh, p.sbo_bh);
  const uint64_t d_b2b = make_bdesc(sb + p.off_bh + (uint32_t)(H / 2 / 8) * p.sbo_bh, p.sbo_bh);

  // predict: the rows of the slot's next tile are bulk-copied (TMA engine) into
  // a per-slot shared-memory buffer one tile ahead; partial tiles, or an
  // x pointer that is not 16-byte aligned, read global memory directly
  uint8_t* xs = smem + p.smem_x + s * p.x_tile_bytes;
  uint64_t* xbar = &bars[9 + s];
  uint32_t phx = 0;
  uint64_t x_next = 0;  // tile whose rows the next phase-0 issue prefetches
  auto x_full = [&](uint64_t tl_) { return p.x_tma != 0u && p.begin + (tl_ + 1) * TILE_M <= p.end; };
  auto x_issue = [&](uint64_t tl_) {  // one thread
    if (tl_ < p.num_tiles && x_full(tl_)) {
      mbar_arrive_expect_tx(xbar, p.x_tile_bytes);
      bulk_g2s(xs, reinterpret_cast<const uint8_t*>(p.x + (p.begin + tl_ * TILE_M) * p.P), p.x_tile_bytes, xbar);
    }
  };
  auto a0_pred = [&](uint64_t tl_, uint64_t I_, A0Regs& a) {
    if (x_full(tl_)) {
      mbar_wait(xbar, phx);
      phx ^= 1u;
      make_a0_row<PREC, true>(p, reinterpret_cast<const float*>(xs) + row * p.P, a);
    } else {
      make_a0_predict<PREC>(p, I_ < p.end ? I_ : p.begin, a);
    }
  };

  // ensemble members >= 1: the slot's tile of the fp32 accumulator is bulk-copied
  // into a per-slot double buffer when the tile's L1 is issued, and read when
  // the tile's prediction is final (~3k cycles later: the HBM latency is hidden)
  uint8_t* accb = smem + p.smem_acc + s * 2 * TILE_M * 4;
  uint32_t pha = 0;  // parity bits of the two buffers' barriers
  auto acc_full = [&](uint64_t tl_) {
    return ENS && p.acc_tma != 0u && p.acc_mode >= 2 && p.begin + (tl_ + 1) * TILE_M <= p.end;
  };
  auto acc_issue = [&](uint64_t tl_, uint32_t b) {  // one thread
    if (tl_ < p.num_tiles && acc_full(tl_)) {
      mbar_arrive_expect_tx(&bars[32 + 2 * s + b], TILE_M * 4);
      bulk_g2s(accb + b * TILE_M * 4, p.t_acc + (p.begin + tl_ * TILE_M - p.acc_base), TILE_M * 4, &bars[32 + 2 * s + b]);
    }
  };
  auto acc_get = [&](uint64_t tl_, uint32_t b, bool valid, uint64_t I_) -> float {
    if (acc_full(tl_)) {
      mbar_wait(&bars[32 + 2 * s + b], (pha >> b) & 1u);
      pha ^= 1u << b;
      return reinterpret_cast<const float*>(accb + b * TILE_M * 4)[row];
    }
    return ens_prefetch(p, valid, I_);
  };
  uint64_t acc_next = 0;  // tile whose accumulator the next phase-0 issue prefetches
  uint32_t acc_buf = 0;   // ... and its buffer

  // every warp of the slot is done with its TMEM writes/reads -> issue one phase
  auto issue = [&](int phase) {
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (issuer) {
      tc_fence_after();
      if (elect_one()) {
        if (phase == 0) {
          if (PRED) x_issue(x_next);  // the A0 tile holds the rows now: the buffer is free
          if (ENS) acc_issue(acc_next, acc_buf);
          if (C::A0_SMEM) umma_f16_ss(dslot, d_a0, d_b1, idesc_full, 0u);
          else umma_f16_ts(dslot, tmem_base + C::A0_COL + 8 * s, d_b1, idesc_full, 0u);
        } else {
          const uint64_t bd = phase == 1 ? d_b2a : d_b2b;
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk) umma_f16_ts(dslot + H / 2, dslot + kk * 8, bd + kk * 16, idesc_half, kk > 0);
          if (C::A0_SMEM) umma_f16_ss(dslot + H / 2, d_ones, bd + (H / 16) * 16, idesc_half, 1u);
          else umma_f16_ts(dslot + H / 2, ones, bd + (H / 16) * 16, idesc_half, 1u);
        }
        umma_commit(&bars[4 + s]);
      }
      __syncwarp();
    }
  };

  uint64_t tile = (uint64_t)blockIdx.x * C::NSLOT + s;
  uint64_t I = p.begin + tile * TILE_M + row;
  const uint64_t dI = (uint64_t)p.dTiles * TILE_M;
  uint32_t D[MAXG];
  if (!PRED) init_digits_n<NG>(p.R, I, D);
  uint32_t phd = 0;
  mbar_wait(&bars[0], 0);

  A0Regs a0;
  if (PRED && issuer && elect_one()) x_issue(tile);
  __syncwarp();
  x_next = tile + p.dTiles;
  acc_next = tile;
  acc_buf = 0;
  if (tile < p.num_tiles) {
    if (PRED) a0_pred(tile, I, a0);
    else if (SPG == 4) make_a0_sweep4(p, slut, D, a0);
    else make_a0_sweep<PREC>(p, slut, D, a0);
    if (!PRED) a0_dump<false>(p, mode, a0, I);
    put_a0(a0);
    if (!C::A0_SMEM) tmem_wait_st();
    issue(0);  // L1 of the first tile
  }
  uint32_t jr = 0;
  for (; tile < p.num_tiles; tile += p.dTiles, ++jr) {
    const bool valid = I < p.end;
    if (ENS) {
      acc_next = tile + p.dTiles;  // the next phase-0 issue starts the next tile
      acc_buf = (jr + 1) & 1u;
    }
    const uint64_t In = I + dI;
    const bool has_next = tile + p.dTiles < p.num_tiles;
    const bool tr = wq == 0 && lane == 0;
    if (tr) trace_ev(p, s, jr, 0);

    float t;
    if (p.NL == 1) {
      mbar_wait(&bars[4 + s], phd);
      phd ^= 1u;
      tc_fence_after();
      t = final_partial<H>(p, dcol, 0);
      if (has_next) {
        if (PRED) {
          a0_pred(tile + p.dTiles, In, a0);
          x_next = tile + 2 * (uint64_t)p.dTiles;
        }
        else {
          odometer_step_n<NG>(p.R, p.dD, D);
          if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC>(p, slut, D, a0);
          a0_dump<false>(p, mode, a0, In);
        }
        put_a0(a0);
        if (!C::A0_SMEM) tmem_wait_st();
        issue(0);
      }
    } else {
      // ---- L1 done -> epi1 in place
      mbar_wait(&bars[4 + s], phd);
      phd ^= 1u;
      tc_fence_after();
      if (tr) trace_ev(p, s, jr, 1);
#pragma unroll
      for (int c = 0; c < H / 32; c += 2) {
        uint32_t v[2][32];
        tmem_ld32(dcol + c * 32, v[0]);
        if (H / 32 > 1) tmem_ld32(dcol + (c + 1) * 32, v[1]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && H / 32 == 1) break;
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = relu_pk16<PREC>(__uint_as_float(v[u][2 * j]), __uint_as_float(v[u][2 * j + 1]));
          tmem_st16(dcol + (c + u) * 16, pk);
        }
      }
      tmem_wait_st();
      if (tr) trace_ev(p, s, jr, 2);
      issue(1);  // L2a: A1 ready
      // ---- L2a done -> load the first half, release it to L2b, then compute
      mbar_wait(&bars[4 + s], phd);
      phd ^= 1u;
      tc_fence_after();
      if (tr) trace_ev(p, s, jr, 3);
      uint32_t v[64];
      final_load<H / 2>(dcol + H / 2, v);
      issue(2);  // L2b: D[H/2, H) consumed
      const float pa = final_compute<H / 2>(p, v, 0);
      if (tr) trace_ev(p, s, jr, 4);
      // ---- next tile's A0 while L2b runs (its 8-column area is idle now)
      if (has_next) {
        if (PRED) {
          a0_pred(tile + p.dTiles, In, a0);
          x_next = tile + 2 * (uint64_t)p.dTiles;
        }
        else {
          odometer_step_n<NG>(p.R, p.dD, D);
          if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC>(p, slut, D, a0);
          a0_dump<false>(p, mode, a0, In);
        }
        put_a0(a0);
      }
      // ---- L2b done -> load the second half, start the next tile's L1, then compute
      mbar_wait(&bars[4 + s], phd);
      phd ^= 1u;
      tc_fence_after();
      if (tr) trace_ev(p, s, jr, 5);
      final_load<H / 2>(dcol + H / 2, v);
      if (has_next) {
        if (!C::A0_SMEM) tmem_wait_st();
        issue(0);  // next tile's L1: A0 stored and all of D read
      }
      const float pb = final_compute<H / 2>(p, v, H / 2);
      if (tr) trace_ev(p, s, jr, 6);
      t = pa + pb;
    }
    t += p.c_out;
    // (accumulator staged in shared memory since the tile's L1 issue: the
    // 128-register budget of the 4-slot kernel has no room to carry it)
    if (!ens_stage(p, valid, I, t, ENS ? acc_get(tile, jr & 1u, valid, I) : ens_prefetch(p, valid, I))) {
    } else if (mode == MODE_TOPK) {
      topk_offer(ts, mycand, ncand, valid, t, I, p.k, lane);
    } else if (valid && mode != MODE_A0) {
      p.t_dense[I - p.begin] = t;
    }
    if (tr) trace_ev(p, s, jr, 7);
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
