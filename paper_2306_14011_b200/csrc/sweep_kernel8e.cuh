// K1 for ensembles (BASELINE cfg 4: E FCNNs averaged per
// config, G15) in ONE pass: every config is decoded once and run through all
// E members, with no HBM accumulator.
//
// The E member images (8 x 41 KB for 17-128-128-1, device feature folded into
// b_1) do not fit one SM's shared memory, so a cluster of two CTAs shares them:
// CTA rank r holds members [r GM, (r+1) GM) resident (GM = E / 2) and both CTAs
// of the pair sweep the SAME tiles (same decoder state, same A0).  Each slot
// runs its tile through its GM members back to back — the A0 tile stays in
// shared memory across them, only the weight descriptors change — with the
// schedule of sweep_kernel8 (final layer pipelined across the units
// (tile, member)).  Tiles alternate between the ranks as the one that
// finishes them: on even tiles rank 1 sends its GM per-member predictions of a
// row to rank 0 with one st.async (16 bytes, completing on rank 0's mbarrier),
// on odd tiles rank 0 sends its ordered partial sum to rank 1; the receiver
// continues the sum in member order e = 0 .. E-1 (the summation order of the
// multi-pass path and of predict, so t is bitwise the same), divides by E and
// runs the top-k.  Per slot, exchange buffer b carries the tiles rank b
// finishes (full: on rank b, tx-counted; empty: on the sender, arrived
// remotely by rank b).
#pragma once
#include "sweep_kernel8.cuh"

namespace surr {

// final-layer FFMA2 steps with member mi's weights w' = y_scale w / 2 from the
// parameter bank (p.ens_w).  mi is a compile-time constant at every call (the
// member loop is unrolled and the CTA rank selects between two calls), so the
// weights are uniform LDCU.128 operands as in the single-net kernel; with a
// run-time member index they compiled to per-thread LDC (-3.7 %), and from the
// shared-memory image as broadcast LDS.128 they cost 11 % (same-box A/B,
// DESIGN section 7).  The accumulator order is final_compute's, so t is
// bitwise the single-net path's.
template <int NC>
__device__ __forceinline__ float final_compute_k(const KParams& p, uint32_t mi, const uint32_t (&v)[64], int n0) {
  uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int j = 0; j < NC; j += 2) {
    const uint64_t w2 = pack2(p.ens_w[mi][n0 + j], p.ens_w[mi][n0 + j + 1]);
    const float x0 = __uint_as_float(v[j]), x1 = __uint_as_float(v[j + 1]);
    acc[(j >> 1) & 1] = ffma2(w2, pack2(x0, x1), acc[(j >> 1) & 1]);
    acc[2 + ((j >> 1) & 1)] = ffma2(w2, pack2(fabsf(x0), fabsf(x1)), acc[2 + ((j >> 1) & 1)]);
  }
  return fin_sum(acc);
}
template <int H, int SPG, int PREC, int GM>
__global__ void __launch_bounds__(512, 1) sweep_kernel8e(const __grid_constant__ KParams p, int mode) {
  constexpr int NG = K0 / SPG;
  constexpr int NSLOT = 4;
  static_assert(H == 128 && GM >= 1 && GM <= 4, "four 128-column slots, up to 4 members per CTA");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = blockIdx.x >> 1;

  // bars: [0] load, [4 + s] slot s MMAs, [32 + 2s + b] exchange full (on rank b),
  // [40 + 2s + b] exchange empty (on rank 1 - b)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);
  float4* xbuf = reinterpret_cast<float4*>(smem + p.smem_x);  // [slot][2][128 rows]
  constexpr uint32_t XBYTES = TILE_M * 16;

  // ---- setup: this rank's GM member images + the value table
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[4 + s], 1);
      for (int i = 0; i < 2 * NSLOT; ++i) {
        mbar_init(&bars[32 + i], 1);
        mbar_init(&bars[40 + i], 1);
      }
      fence_mbar_init();
      fence_proxy_async_smem();
      const uint32_t wbytes = GM * p.w_bytes;
      const uint8_t* wsrc = (const uint8_t*)p.w_gmem + (size_t)rank * wbytes;
      mbar_arrive_expect_tx(&bars[0], wbytes + p.lut_bytes);
      for (uint32_t off = 0; off < wbytes; off += 32768u)
        bulk_g2s(smem + off, wsrc + off, min(32768u, wbytes - off), &bars[0]);
      if (p.lut_bytes) bulk_g2s(smem + p.smem_lut, p.lut_gmem, p.lut_bytes, &bars[0]);
      // arm the first use of every exchange buffer this CTA receives (b = rank)
      for (int i = 0; i < 2 * NSLOT; ++i)
        if ((uint32_t)(i & 1) == rank) mbar_arrive_expect_tx(&bars[32 + i], XBYTES);
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
  if (warp < 4) {  // the bias ones block of the layer-2 bias K step
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = one16<PREC>();
    st_a0_smem(smem + p.smem_ones, warp * 32u + lane, ones);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised (and armed) before any remote operation
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // ================= slot warpgroups (self-issuing) =================
  const uint32_t s = warp >> 2;
  const uint32_t wq = warp & 3u;
  const uint32_t row = wq * 32u + lane;
  const uint32_t dslot = tmem_base + s * H;
  const uint32_t dcol = dslot + ((wq * 32u) << 16);
  uint8_t* a0tile = smem + p.smem_a0 + s * 4096u;
  const uint8_t* slut = smem + p.smem_lut;
  surr_record* mycand = ts.cand + (size_t)warp * CAND_CAP;
  uint32_t ncand = 0;
  const uint32_t bar_id = 1 + s;
  const uint32_t sb = smem_u32(smem);
  const uint64_t d_ones = make_bdesc(sb + p.smem_ones, 256);
  const uint64_t d_a0 = make_bdesc(sb + p.smem_a0 + s * 4096u, 256);
  const uint32_t idesc_full = p.idesc;
  const uint32_t idesc_half = (p.idesc & ~(0x3Fu << 17)) | (((uint32_t)(H / 2) >> 3) << 17);
  // member m's image starts m w_bytes into shared memory: descriptor start
  // addresses advance by (m w_bytes) >> 4 (addresses < 256 KB: no carry out)
  const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
  const uint64_t d_b2a = make_bdesc(sb + p.off_bh, p.sbo_bh);
  const uint64_t d_b2b = make_bdesc(sb + p.off_bh + (uint32_t)(H / 2 / 8) * p.sbo_bh, p.sbo_bh);
  const uint64_t d_step = (uint64_t)(p.w_bytes >> 4);

  auto issue = [&](int phase, uint32_t m) {
    tc_fence_before();
    named_bar_sync(bar_id, 128);
    if (wq == 0) {
      tc_fence_after();
      if (elect_one()) {
        if (phase == 0) {
          umma_f16_ss(dslot, d_a0, d_b1 + m * d_step, idesc_full, 0u);
        } else {
          const uint64_t bd = (phase == 1 ? d_b2a : d_b2b) + m * d_step;
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk) umma_f16_ts(dslot + H / 2, dslot + kk * 8, bd + kk * 16, idesc_half, kk > 0);
          umma_f16_ss(dslot + H / 2, d_ones, bd + (H / 16) * 16, idesc_half, 1u);
        }
        umma_commit(&bars[4 + s]);
      }
      __syncwarp();
    }
  };
  auto store_a0 = [&](const uint32_t (&D)[MAXG], uint64_t Ir) {
    A0Regs a0;
    if (SPG == 4) make_a0_sweep4(p, slut, D, a0); else make_a0_sweep<PREC>(p, slut, D, a0);
    if (rank == 0) a0_dump<false>(p, mode, a0, Ir);
    st_a0_smem(a0tile, row, a0.hi);
    fence_proxy_async_smem();
  };

  // per-tile member predictions: each rank keeps its members' running sum in
  // member order and the values themselves.  The tiles alternate between the
  // ranks as the one that finishes them (sums, divides by E, runs the top-k):
  // exchange buffer b = tseq & 1 always flows towards rank b, so the finishing
  // work and the release / acquire handshakes are split evenly between the two
  // CTAs (rank 1 used to idle on rank 0's handshake).  Rank 1 sends its GM
  // values, rank 0 its ordered partial sum; the receiver continues the sum in
  // member order e = 0 .. E-1 either way (bitwise the multi-pass order).
  float tsum = 0.0f;
  float tm[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  uint32_t tseq = 0;  // tiles completed by this slot
  // unit (tile, member m) is final: t_m = dot + c_m; on the tile's last member,
  // exchange and (receiver) emit
  auto unit_done = [&](float dot, uint32_t m, uint64_t Ir) {
    const float t = dot + p.ens_c[rank * GM + m];
    tsum = m == 0 ? t : tsum + t;
#pragma unroll
    for (int i = 0; i < GM; ++i) tm[i] = (uint32_t)i == m ? t : tm[i];  // (registers, not a local array)
    if (m + 1 < GM) return;
    const uint32_t b = tseq & 1u, q = tseq >> 1;
    float4* xb = xbuf + (s * 2 + b) * TILE_M;
    if (rank != b) {  // sender: buffer b's previous use has been read by rank b
      mbar_wait_cluster(&bars[40 + 2 * s + b], (q & 1u) ^ 1u);
      if (rank == 1) st_async_v4(&xb[row], tm[0], tm[1], tm[2], tm[3], &bars[32 + 2 * s + b], 0);
      else st_async_v4(&xb[row], tsum, 0.0f, 0.0f, 0.0f, &bars[32 + 2 * s + b], 1);
    } else {
      mbar_wait_cluster(&bars[32 + 2 * s + b], q & 1u);
      const float4 u = xb[row];
      float acc;
      if (rank == 0) {  // members GM .. 2 GM - 1 after this CTA's ordered partial
        acc = tsum;
        const float uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < GM; ++i) acc = acc + uu[i];
      } else {  // rank 0's ordered partial, then this CTA's members in order
        acc = u.x;
#pragma unroll
        for (int i = 0; i < GM; ++i) acc = acc + tm[i];
      }
      const float tt = acc * p.inv_e;
      named_bar_sync(bar_id, 128);  // every row of the buffer read
      if (wq == 0 && lane == 0) {
        mbar_arrive_expect_tx(&bars[32 + 2 * s + b], XBYTES);  // arm its next use
        mbar_arrive_cluster(&bars[40 + 2 * s + b], rank ^ 1u);  // and hand it back to the sender
      }
      const bool valid = Ir < p.end;
      if (mode == MODE_TOPK) topk_offer(ts, mycand, ncand, valid, tt, Ir, p.k, lane);
      else if (valid && mode == MODE_DENSE) p.t_dense[Ir - p.begin] = tt;
    }
    ++tseq;
  };

  const uint32_t npairs = gridDim.x >> 1;
  uint64_t tile = (uint64_t)pair * NSLOT + s;
  uint64_t I = p.begin + tile * TILE_M + row;
  const uint64_t dI = (uint64_t)p.dTiles * TILE_M;  // dTiles = NSLOT * npairs
  (void)npairs;
  uint32_t D[MAXG];
  init_digits_n<NG>(p.R, I, D);
  uint32_t ph = 0;
  mbar_wait(&bars[0], 0);
  if (tile < p.num_tiles) {
    store_a0(D, I);
    issue(0, 0);  // L1 of the first unit
  }
  // the previous unit's dot product (its half a + half b) and identity
  float pdot = 0.0f;
  uint32_t pm = 0;
  uint64_t pI = 0;
  bool carry = false;
  for (; tile < p.num_tiles; tile += p.dTiles) {
    const uint64_t In = I + dI;
    const bool has_next = tile + p.dTiles < p.num_tiles;
#pragma unroll  // compile-time member index: uniform final-layer weight operands
    for (uint32_t m = 0; m < (uint32_t)GM; ++m) {
      const bool last_m = m + 1 == (uint32_t)GM;
      // ---- L1(unit) done -> epilogue 1 in place
      mbar_wait(&bars[4 + s], ph);
      ph ^= 1u;
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < H / 32; ++c) {  // 32 columns per TMEM wait (register budget)
        uint32_t v[32];
        tmem_ld32(dcol + c * 32, v);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = relu_pk16<PREC>(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        tmem_st16(dcol + c * 16, pk);
      }
      tmem_wait_st();
      issue(1, m);  // L2a
      // ---- L2a shadow: finish the previous unit; after the tile's last L1, the next tile's A0
      if (carry) unit_done(pdot, pm, pI);
      if (last_m && has_next) {
        odometer_step_n<NG>(p.R, p.dD, D);
        store_a0(D, In);
      }
      // ---- L2a done: half a, L2b
      mbar_wait(&bars[4 + s], ph);
      ph ^= 1u;
      tc_fence_after();
      float pa;
      {
        uint32_t v[64];
        final_load<H / 2>(dcol + H / 2, v);
        issue(2, m);
        // (blockIdx.x & 1 = this CTA's rank in its cluster of two, members rank GM + m)
        pa = (blockIdx.x & 1u) ? final_compute_k<H / 2>(p, GM + m, v, 0) : final_compute_k<H / 2>(p, m, v, 0);
      }
      // ---- L2b done: half b, next unit's L1 (same A0 with the next member, or the next tile's)
      mbar_wait(&bars[4 + s], ph);
      ph ^= 1u;
      tc_fence_after();
      {
        uint32_t v[64];
        final_load<H / 2>(dcol + H / 2, v);
        if (!last_m) issue(0, m + 1);
        else if (has_next) issue(0, 0);
        pdot = pa + ((blockIdx.x & 1u) ? final_compute_k<H / 2>(p, GM + m, v, H / 2) : final_compute_k<H / 2>(p, m, v, H / 2));
      }
      pm = m;
      pI = I;
      carry = true;
    }
    I = In;
  }
  if (carry) unit_done(pdot, pm, pI);
  if (mode == MODE_TOPK) topk_post(ts, mycand, ncand, lane);

  // ---- teardown (each CTA's list holds the tiles it finished)
  tc_fence_before();
  __syncthreads();
  if (mode == MODE_TOPK) {
    topk_drain(ts, p.k, warp, lane);
    __syncthreads();
    const surr_record* L = ts.lists + (size_t)ts.misc[1] * p.k;
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) p.recs[(size_t)blockIdx.x * p.k + i] = L[i];
  }
  cluster_sync();  // no exchange traffic left in flight towards either CTA
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  grid_merge_tail(p, mode, smem);
}

}  // namespace surr
