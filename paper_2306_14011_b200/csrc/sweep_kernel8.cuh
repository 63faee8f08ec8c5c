// K1, 16-bit variant (FP16 / BF16) for 14-128-128-1 sweeps (cfg2, cfg5, the
// paper's space), with the final layer software-pipelined across tiles.
// Same warps (four self-issuing slots of one warpgroup, 128-row tiles), TMEM
// layout and arithmetic as sweep_kernel3; what changes is WHEN each warpgroup
// does its FP32 work.
//
// A slot's TMEM region is released only by its own chain
//   L1 -> wake -> epilogue-1 -> L2a -> wake -> load half a -> L2b -> wake ->
//   load half b -> next L1,
// and anything the warps do between two links lengthens it.  sweep_kernel3
// computes the whole second final-layer half and the top-k of tile t between
// "L1(t+1) issued" and "epilogue-1(t+1)" (~1,300 cycles against an L1 of
// ~250), and its next-tile decode plus the first half in the L2b shadow: the
// chain is ~3,700 cycles for 640 tensor cycles (a CTA timeline, ncu 68.6 %
// tensor-pipe activity).  Here each piece of FP32 work sits in the shadow of
// an MMA the slot is waiting for anyway:
//
//   L1(t)  shadow : FP32 final layer over half b(t-1) (CB = 0, the default;
//                   CB = 16 leaves its last 16 columns for the L2a shadow)
//   epilogue-1(t) : (on the chain) ReLU + pack of D1(t)
//   L2a(t) shadow : t(t-1) (+ the carried columns), top-k, decode + store
//                   A0(t+1) (L1(t) has consumed the A0 tile)
//   L2b(t) shadow : FP32 final layer over half a(t)
//
// so tile t-1's prediction (or, CB > 0, half b's accumulators and its last CB
// columns) is carried into tile t in registers, and the last tile is finished
// after the loop.  The FFMA2 order per accumulator is final_compute's, so t is
// bitwise the 4-slot kernel's (and the explicit-batch predict path's).
// Measured (same box, cfg2 / cfg5 evals/s): 3.49e10 / 3.15e10 against
// sweep_kernel3's 3.35e10 / 2.97e10; ncu tensor-pipe activity stays ~69 %
// (the final-layer FP32 work, ~470 warp instructions per warp and tile, still
// exceeds the MMA shadows: sweep_kernel3.cuh / DESIGN.md section 6).
#pragma once
#include "sweep_kernel3.cuh"

namespace surr {

// final-layer FFMA2 steps over NC columns held in registers v[0..NC), output
// neurons n0 .. n0+NC-1, into acc (the accumulator order of final_compute, so
// a half computed in two pieces is bitwise the half computed at once)
template <int NC>
__device__ __forceinline__ void fin_acc(const KParams& p, const uint32_t* v, int n0, uint64_t (&acc)[4]) {
#pragma unroll
  for (int j = 0; j < NC; j += 2) relu_dot2(p, v[j], v[j + 1], n0 + j, acc, j);
}
__device__ __forceinline__ float fin_sum(const uint64_t (&acc)[4]) {
  float a8[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
  return ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
}

// CB: columns of half b carried into the next iteration (16: the 48 others in
// the L1 shadow; 0: all of half b in the L1 shadow, so the epilogue can load
// 64 columns per TMEM wait within the register budget)
// FM: the mode fixed at compile time (MODE_TOPK: the sweep itself, no dense /
// operand-dump code or per-tile mode tests), or -1 (any mode, at run time)
template <int H, int SPG, int PREC, int CB = 16, int FM = -1>
__global__ void __launch_bounds__(512, 1) sweep_kernel8(const __grid_constant__ KParams p, int mode_rt) {
  const int mode = FM >= 0 ? FM : mode_rt;
  constexpr int EC = CB == 0 ? 2 : 1;  // 32-column chunks per TMEM load wait in epilogue 1
  // SPG = 0: the explicit-batch (predict) instantiation: rows from HBM instead
  // of the decoder (bulk-copied one tile ahead into a per-slot staging buffer)
  constexpr bool PRED = SPG == 0;
  constexpr int NG = PRED ? 1 : K0 / SPG;
  constexpr int NSLOT = 4;
  static_assert(H == 128, "four 128-column slots");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);  // [0] load, [4 + s] slot s
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[4 + s], 1);
      if (PRED)
        for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[9 + s], 1);  // row staging
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint32_t lutb = PRED ? 0u : p.lut_bytes;
      mbar_arrive_expect_tx(&bars[0], p.w_bytes + lutb);
      for (uint32_t off = 0; off < p.w_bytes; off += 32768u)
        bulk_g2s(smem + off, (const uint8_t*)p.w_gmem + off, min(32768u, p.w_bytes - off), &bars[0]);
      if (lutb) bulk_g2s(smem + p.smem_lut, p.lut_gmem, lutb, &bars[0]);
    }
    __syncwarp();
    tmem_alloc<512>(tmem_slot);
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
  if (warp < 4) {  // the bias ones block (row-constant [1, 0, ...]) of the layer-2 bias K step
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = one16<PREC>();
    st_a0_smem(smem + p.smem_ones, warp * 32u + lane, ones);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // ================= slot warpgroups (self-issuing) =================
  const uint32_t s = warp >> 2;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t dslot = tmem_base + s * H;                 // lane 0 view (UMMA operands)
  const uint32_t dcol = dslot + ((wq * 32u) << 16);          // this warp's lanes
  // this row's place in the slot's A0 tile (K-major core matrices, st_a0_smem's layout)
  const uint32_t a0_st = smem_u32(smem + p.smem_a0 + s * 4096u) + (row >> 3) * 256u + (row & 7u) * 16u;
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)warp * CAND_CAP;
  uint32_t ncand = 0;
  const uint32_t bar_id = 1 + s;
  const uint32_t sb = smem_u32(smem);
  const uint64_t d_ones = make_bdesc(sb + p.smem_ones, 256);
  const uint64_t d_a0 = make_bdesc(sb + p.smem_a0 + s * 4096u, 256);
  const uint32_t idesc_full = p.idesc;
  const uint32_t idesc_half = (p.idesc & ~(0x3Fu << 17)) | (((uint32_t)(H / 2) >> 3) << 17);
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint64_t d_b2a = make_bdesc(sb + p.off_bh, p.sbo_bh);
  const uint64_t d_b2b = make_bdesc(sb + p.off_bh + (uint32_t)(H / 2 / 8) * p.sbo_bh, p.sbo_bh);

  // predict: the rows of the slot's next tile are bulk-copied (TMA engine) into
  // a per-slot shared-memory buffer one tile ahead (issued with the L1 that
  // frees it); partial tiles, or an x pointer that is not 16-byte aligned,
  // read global memory directly (sweep_kernel3's prologue)
  uint8_t* xs = smem + p.smem_x + s * p.x_tile_bytes;
  uint64_t* xbar = &bars[9 + s];
  uint32_t phx = 0;
  uint64_t x_next = 0;  // tile whose rows the next L1 issue prefetches
  auto x_full = [&](uint64_t tl_) { return p.x_tma != 0u && p.begin + (tl_ + 1) * TILE_M <= p.end; };
  auto x_issue = [&](uint64_t tl_) {  // one thread
    if (tl_ < p.num_tiles && x_full(tl_)) {
      mbar_arrive_expect_tx(xbar, p.x_tile_bytes);
      bulk_g2s(xs, reinterpret_cast<const uint8_t*>(p.x + (p.begin + tl_ * TILE_M) * p.P), p.x_tile_bytes, xbar);
    }
  };

  // every warp of the slot is done with its TMEM writes / reads and A0 stores
  // -> one elected lane issues the phase (0: L1, 1: L2a, 2: L2b) and commits
  auto issue = [&](int phase) {
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (wq == 0) {
      tc_fence_after();
      if (elect_one()) {
        if (phase == 0) {
          if (PRED) x_issue(x_next);  // the A0 tile holds the rows now: the buffer is free
          umma_f16_ss(dslot, d_a0, d_b1, idesc_full, 0u);
        } else {
          const uint64_t bd = phase == 1 ? d_b2a : d_b2b;
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk) umma_f16_ts(dslot + H / 2, dslot + kk * 8, bd + kk * 16, idesc_half, kk > 0);
          umma_f16_ss(dslot + H / 2, d_ones, bd + (H / 16) * 16, idesc_half, 1u);
        }
        umma_commit(&bars[4 + s]);
      }
      __syncwarp();
    }
  };
  // the layer-1 operand row of tile tl_ (index Ir): decoded, or (PRED) the row's raw values
  auto store_a0 = [&](const uint32_t (&D)[MAXG], uint64_t tl_, uint64_t Ir) {
    A0Regs a0;
    if constexpr (PRED) {
      if (x_full(tl_)) {
        mbar_wait(xbar, phx);
        phx ^= 1u;
        make_a0_row<PREC, true>(p, reinterpret_cast<const float*>(xs) + row * p.P, a0);
      } else {
        make_a0_predict<PREC>(p, Ir < p.end ? Ir : p.begin, a0);
      }
    } else {
      if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC>(p, slut, D, a0);
    }
    if (FM != MODE_TOPK && !PRED) a0_dump<false>(p, mode, a0, Ir);
    st_shared_v4(a0_st, a0.hi[0], a0.hi[1], a0.hi[2], a0.hi[3]);
    st_shared_v4(a0_st + 128u, a0.hi[4], a0.hi[5], a0.hi[6], a0.hi[7]);
    fence_proxy_async_smem();
  };
  // a tile's prediction is final: top-k / dense output
  auto emit = [&](float t, uint64_t Ir) {
    const bool valid = Ir < p.end;
    if (mode == MODE_TOPK) topk_offer(ts, mycand, ncand, valid, t, Ir, p.k, lane);
    else if (valid && (mode == MODE_DENSE || mode == MODE_PREDICT)) p.t_dense[Ir - p.begin] = t;
  };

  uint64_t tile = (uint64_t)blockIdx.x * NSLOT + s;
  uint64_t I = p.begin + tile * TILE_M + row;
  const uint64_t dI = (uint64_t)p.dTiles * TILE_M;
  uint32_t D[MAXG];
  if (!PRED) init_digits_n<NG>(p.R, I, D);
  uint32_t ph = 0;
  mbar_wait(&bars[0], 0);
  if (PRED) {
    if (wq == 0 && elect_one()) x_issue(tile);
    __syncwarp();
    x_next = tile + p.dTiles;
  }
  if (tile < p.num_tiles) {
    store_a0(D, tile, I);
    issue(0);  // L1 of the first tile
  }
  // tile t-1 carried into iteration t: half a's sum, half b's accumulators
  // after its first 32 columns, and its last 32 columns
  float pa = 0.0f;
  uint64_t accb[4];
  uint32_t vb[CB > 0 ? CB : 1];
  bool carry = false;
  uint32_t jr = 0;
  const bool tr = wq == 0 && lane == 0;
  for (; tile < p.num_tiles; tile += p.dTiles, ++jr) {
    const uint64_t In = I + dI;
    const bool has_next = tile + p.dTiles < p.num_tiles;
    if (tr) trace_ev(p, s, jr, 0);
    // ---- L1(t) done -> epilogue 1 in place, two 32-column chunks per wait (chunk c is
    // read before packed chunk c goes to columns 16c .. 16c+15, already read)
    mbar_wait(&bars[4 + s], ph);
    ph ^= 1u;
    tc_fence_after();
    if (tr) trace_ev(p, s, jr, 1);
#pragma unroll
    for (int c = 0; c < H / 32; c += EC) {
      uint32_t v[EC][32];
#pragma unroll
      for (int u = 0; u < EC; ++u) tmem_ld32(dcol + (c + u) * 32, v[u]);
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pk[j] = relu_pk16<PREC>(__uint_as_float(v[u][2 * j]), __uint_as_float(v[u][2 * j + 1]));
        tmem_st16(dcol + (c + u) * 16, pk);
      }
    }
    tmem_wait_st();
    issue(1);  // L2a
    if (tr) trace_ev(p, s, jr, 2);
    // ---- L2a shadow: finish tile t-1, decode + store A0(t+1)
    if (carry) {
      if (CB > 0) {
        fin_acc<CB>(p, vb, H - CB, accb);
        emit((pa + fin_sum(accb)) + p.c_out, I - dI);
      } else {
        emit(pa + p.c_out, I - dI);
      }
    }
    if (has_next) {
      if (!PRED) odometer_step_n<NG>(p.R, p.dD, D);
      store_a0(D, tile + p.dTiles, In);
      if (PRED) x_next = tile + 2 * (uint64_t)p.dTiles;
    }
    if (tr) trace_ev(p, s, jr, 3);
    // ---- L2a done: load half a, release it to L2b, FP32 half a in the L2b shadow
    mbar_wait(&bars[4 + s], ph);
    ph ^= 1u;
    tc_fence_after();
    if (tr) trace_ev(p, s, jr, 4);
    {
      uint32_t v[64];
      final_load<H / 2>(dcol + H / 2, v);
      issue(2);  // L2b
      pa = final_compute<H / 2>(p, v, 0);
    }
    if (tr) trace_ev(p, s, jr, 5);
    // ---- L2b done: load half b, start L1(t+1), FP32 over its first 32 columns
    mbar_wait(&bars[4 + s], ph);
    ph ^= 1u;
    tc_fence_after();
    if (tr) trace_ev(p, s, jr, 6);
    {
      uint32_t v[64];
      final_load<H / 2>(dcol + H / 2, v);
      if (has_next) issue(0);
#pragma unroll
      for (int j = 0; j < 4; ++j) accb[j] = 0ull;
      fin_acc<H / 2 - CB>(p, v, H / 2, accb);
#pragma unroll
      for (int j = 0; j < CB; ++j) vb[j] = v[H / 2 - CB + j];
      if (CB == 0) pa += fin_sum(accb);  // nothing left of half b: carry t - c_out only
    }
    carry = true;
    if (tr) trace_ev(p, s, jr, 7);
    I = In;
  }
  if (carry) {  // the slot's last tile
    if (CB > 0) {
      fin_acc<CB>(p, vb, H - CB, accb);
      emit((pa + fin_sum(accb)) + p.c_out, I - dI);
    } else {
      emit(pa + p.c_out, I - dI);
    }
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
    tmem_dealloc(tmem_base, 512);
  }
  grid_merge_tail(p, mode, smem);
}

}  // namespace surr
