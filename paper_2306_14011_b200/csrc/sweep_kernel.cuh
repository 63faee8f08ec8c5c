// Fused exhaustive-sweep kernel (K1), explicit-batch predict (K3), block
// top-k (a8) and the list merge (K2) for sm_100a.
//
// Per flat config index I:
//   a2  mixed-radix decode on "super digits": group g = parameters 2g, 2g+1
//       (radix R_g = r_2g r_2g+1); each thread keeps the digits of its row in
//       registers and advances them by the constant per-tile index stride with
//       a carry-propagating odometer (no division in the loop);
//   a3  normalisation prologue = one shared-memory lookup per group of the
//       pre-normalised, pre-rounded operand pair (StandardScaler);
//   a4  layer-1 UMMA, K0 = 16 (14 params + ones slot carrying b_1 + 0);
//   a5  hidden epilogue: tcgen05.ld D -> ReLU -> BF16x2 / TF32 hi-lo ->
//       tcgen05.st A (the next layer's A operand lives in TMEM); hidden-layer
//       biases ride in the UMMA as an extra K block against a constant ones
//       block in TMEM when it fits (BIAS_MMA), else are added here;
//   a6  hidden UMMAs, B = weights resident in shared memory (bulk-copied once);
//   a7  final H -> 1 layer in FP32 on CUDA cores (packed FFMA2) + de-standardisation;
//   a8  warp ballot filter against the CTA's k-th best, per-warp candidate
//       buffer, rank-based merge into the CTA's sorted top-k.
//
// CTA roles: warp 0 lane 0 issues every tcgen05.mma (blocking waits, round
// robin over slots); warpgroups 1..NSLOT each own one TMEM slot (D accumulator
// + A operand for a 128-row tile) and run decode, epilogues and top-k for that
// slot's tiles, so NSLOT tiles are in flight and one slot's CUDA-core epilogue
// overlaps the other slot's MMAs.
#pragma once
#include <cstddef>
#include <cstdint>

#include "sm100_ptx.cuh"
#include "../../include/surrogate.h"

namespace surr {

// PREC_FP32 = 3xTF32, PREC_FP32H = 3xFP16 (both the "FP32 path"); PREC_FP16 =
// 1xFP16 hidden layers (same tensor rate as BF16, 3 more mantissa bits)
enum { PREC_BF16 = 0, PREC_FP32 = 1, PREC_TF32 = 2, PREC_FP16 = 3, PREC_FP32H = 4 };
// 16-bit operand kernels (kind::f16): one element per half column
__host__ __device__ constexpr bool is16(int prec) { return prec == PREC_BF16 || prec == PREC_FP16; }
// relu + pack / pack a column pair into the precision's 16-bit operand format
template <int PREC>
__device__ __forceinline__ uint32_t relu_pk16(float lo, float hi) {
  return PREC == PREC_FP16 ? relu_f16x2(lo, hi) : relu_bf16x2(lo, hi);
}
template <int PREC>
__device__ __forceinline__ uint32_t pk16(float lo, float hi) {
  return PREC == PREC_FP16 ? f16x2(lo, hi) : bf16x2(lo, hi);
}
// 1.0 in the precision's 16-bit format (K slot 0 of the bias ones block)
template <int PREC>
__host__ __device__ constexpr uint32_t one16() { return PREC == PREC_FP16 ? 0x3C00u : 0x3F80u; }
// MODE_A0: parity hook of the decoder + value table (a2, a3): the sweep runs as
// in MODE_DENSE but writes, per config, the layer-1 operand row it built
enum { MODE_TOPK = 0, MODE_DENSE = 1, MODE_PREDICT = 2, MODE_A0 = 3 };

constexpr int MAXG = 8;       // super-digit groups = A0 column pairs (K0 / 2)
constexpr int K0 = 16;        // layer-1 K (P + ones slot <= 16)
constexpr int TILE_M = 128;   // rows per tile (UMMA M)
constexpr int CAND_CAP = 64;  // per-warp top-k candidate buffer
constexpr uint32_t KEY_SENT = 0xFFFFFFFFu;
constexpr uint64_t IDX_SENT = ~0ull;

struct KParams {
  // rows
  uint64_t begin, end, num_tiles;
  uint32_t dTiles;           // tile stride of one slot (= NSLOT * gridDim.x)
  // decoder: group g covers A0 slots 2g, 2g+1; groups without parameters have R = 1
  uint32_t R[MAXG];          // group radix
  uint32_t dD[MAXG];         // digits of the per-tile index stride dTiles * 128
  uint32_t lut_off[MAXG];    // first table entry of group g
  const void* lut_gmem;
  uint32_t lut_bytes;
  // predict rows
  const float* x;
  uint32_t P;
  // input map z_j = fma(x_j, zinv_j, zc_j), zinv = fp32(1 / scale), zc = fp32(-shift / scale)
  // (P:273 StandardScaler); the host value table evaluates the same fp32 FMA, so a row
  // predicted from HBM and the same config decoded in a sweep see identical operands
  float zinv[K0];
  float zc[K0];
  // model
  uint32_t NL;               // UMMA layers (= number of hidden layers)
  const void* w_gmem;
  uint32_t w_bytes;
  uint32_t off_b1, off_b1lo, off_bh, stride_bh, lo_delta_h;
  uint32_t off_fin;          // final-layer [w' (H), -b (H)] floats in the shared-memory image
  uint32_t w_rank_stride;    // CTA-pair kernel: bytes between the two ranks' images
  uint32_t sbo_b1, sbo_bh;
  uint32_t idesc;
  float c_out;
  // epilogue constants in the kernel-parameter (constant) bank
  alignas(16) float fin_w[128];  // y_scale * w_out (16-byte aligned: LDCU.128 operand loads)
  alignas(16) float fin_nb[128];  // -b of the last hidden layer (0 when folded into the UMMA)
  alignas(16) float hbias[2][128];  // biases of model layers 2 .. NL-1 (when not folded)
  // outputs
  uint32_t k;
  surr_record* recs;         // MODE_TOPK: gridDim.x * k records
  // fused grid merge (a9 in K1, MODE_TOPK): per-node tickets of the CTA merge
  // tree (null: K2 merges), merged outputs
  uint32_t* done_ctr;
  uint64_t* out_idx;
  float* out_t;
  surr_record* out_recs;
  float* t_dense;            // MODE_DENSE / MODE_PREDICT
  uint32_t* a0_dump;         // MODE_A0: 16 words per sampled config (hi columns, then lo columns)
  uint64_t a0_stride;        // MODE_A0: configs begin, begin + a0_stride, ... are written
  uint32_t smem_lut, smem_lists, smem_cand, smem_misc;  // byte offsets in dynamic smem
  uint32_t smem_a0, smem_ones;  // SS-form A0 tiles / ones block (4-slot kernel)
  uint32_t smem_x, x_tile_bytes, x_tma;  // predict: per-slot staging of a tile's rows (bulk copy)
  // ensemble passes: acc_mode 0 = single net; 1 = first member,
  // t_acc[I - acc_base] = t; 2 = t_acc += t; 3 = last member, t = (t_acc + t) * inv_e
  float* t_acc;
  uint64_t acc_base;
  uint32_t acc_mode;
  float inv_e;
  uint32_t smem_acc, acc_tma;  // 4-slot kernel: per-slot double buffer of a tile's t_acc (bulk copies)
  // single-pass ensemble on CTA pairs (sweep_kernel8e): members per CTA, E,
  // each member's de-standardisation constant, shared-memory weight region
  uint32_t ens_gm, ens_e;
  float ens_c[16];
  alignas(16) float ens_w[8][128];  // members' final-layer w' = y_scale w / 2 (uniform LDCU.128 operands)
  // debug timeline (CTA 0 only): trace[ev] = clock64 of event ev, or null
  unsigned long long* trace;
  uint32_t trace_n;
  uint32_t variant;  // schedule variant (development A/B switch, env SURR_VARIANT; 0 = default)
};

static_assert(offsetof(KParams, fin_w) % 16 == 0 && offsetof(KParams, fin_nb) % 16 == 0 &&
                  offsetof(KParams, ens_w) % 16 == 0,
              "epilogue constants must stay 16-byte aligned in the parameter bank (LDCU.128)");

// Ensemble accumulator value of row I, loaded at the start of a tile so that
// its latency is hidden behind the tile's MMAs (members e >= 1)
__device__ __forceinline__ float ens_prefetch(const KParams& p, bool valid, uint64_t I) {
  return (p.acc_mode >= 2 && valid) ? p.t_acc[I - p.acc_base] : 0.0f;
}
// Ensemble stage of one row's prediction; false = no output in this pass.
// Uniform across a warp (depends on acc_mode only), so ballots stay legal.
__device__ __forceinline__ bool ens_stage(const KParams& p, bool valid, uint64_t I, float& t, float accp) {
  if (p.acc_mode == 0) return true;
  float* a = p.t_acc + (I - p.acc_base);
  if (p.acc_mode == 1) { if (valid) *a = t; return false; }
  if (p.acc_mode == 2) { if (valid) *a = accp + t; return false; }
  t = (accp + t) * p.inv_e;  // members summed in order e = 0 .. E-1, mean in seconds
  return true;
}

// debug timeline of CTA 0: slot s, tile round j, event e -> one clock64 stamp
// (compiled in only with -DSURR_TRACE)
__device__ __forceinline__ void trace_ev(const KParams& p, uint32_t s, uint32_t j, uint32_t e) {
#ifdef SURR_TRACE
  if (p.trace && blockIdx.x == 0) {
    const uint32_t i = (j * 4 + s) * 16 + e;
    if (i < p.trace_n) p.trace[i] = clock64();
  }
#endif
}

template <int PREC, int H>
struct Cfg {
  static constexpr int A_COLS = is16(PREC) ? H / 2 : (PREC == PREC_FP32 ? 2 * H : H);
  static constexpr int SLOT_COLS = H + A_COLS;
  static constexpr int NSLOT = (2 * SLOT_COLS <= 512) ? 2 : 1;
  // hidden-layer biases as an extra UMMA K block against a shared ones block
  static constexpr bool BIAS_MMA = NSLOT * SLOT_COLS + 8 <= 512;
  static constexpr int ONES_COL = NSLOT * SLOT_COLS;
  static constexpr int NEED = NSLOT * SLOT_COLS + (BIAS_MMA ? 8 : 0);
  static constexpr int TMEM_COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 * (1 + NSLOT);
  static constexpr int PASSES_H = PREC == PREC_FP32 ? 3 : 1;   // hidden layers
  static constexpr int PASSES_1 = is16(PREC) ? 1 : 3;   // layer 1
  static constexpr int KSTEP = is16(PREC) ? 16 : 8;     // K per UMMA
  // A0 lo-part column offset (tf32 modes): fp32 keeps lo next to the hidden lo region
  static constexpr int A0_LO = PREC == PREC_FP32 ? H : K0;
  static_assert(NEED <= 512, "TMEM budget");
};

// order-preserving float -> uint32 (NaN after +inf)
__device__ __forceinline__ uint32_t f2key(float t) {
  uint32_t u = __float_as_uint(t);
  if (t != t) return KEY_SENT;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}
__device__ __forceinline__ bool rec_less(uint32_t ka, uint64_t ia, uint32_t kb, uint64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// SMEM matrix descriptor, K-major, SWIZZLE_NONE: core matrices of 8 rows x 16 B;
// LBO = byte distance of K-adjacent core matrices (128), SBO = distance of
// 8-row groups; version 1 (bits 46-47), layout type 0 (bits 61-63).
__device__ __forceinline__ uint64_t make_bdesc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  return d;
}

// ------------------------------------------------------------ a2: decoder
// Super digits of I (group 0 most significant): one u64 division
// per group, done once per thread.  Rows past |S| (masked tail) clamp the top
// digit so every table index stays in range.
__device__ __forceinline__ void init_digits(const uint32_t* R, uint64_t I, uint32_t (&D)[MAXG]) {
#pragma unroll
  for (int g = MAXG - 1; g >= 0; --g) {
    const uint64_t r = R[g];
    D[g] = (uint32_t)(I % r);
    I /= r;
  }
  if (I) D[0] = R[0] - 1u;
}
template <int NG>
__device__ __forceinline__ void init_digits_n(const uint32_t* R, uint64_t I, uint32_t (&D)[MAXG]) {
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    const uint64_t r = R[g];
    D[g] = (uint32_t)(I % r);
    I /= r;
  }
  if (I) D[0] = R[0] - 1u;
}
template <int NG>
__device__ __forceinline__ void odometer_step_n(const uint32_t* R, const uint32_t* dD, uint32_t (&D)[MAXG]) {
  uint32_t carry = 0;
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    const uint32_t d = D[g] + dD[g] + carry;
    carry = d >= R[g] ? 1u : 0u;
    D[g] = carry ? d - R[g] : d;
  }
}
// D <- digits of (I + stride) mod |S|: add the stride's digits with carries.
__device__ __forceinline__ void odometer_step(const uint32_t* R, const uint32_t* dD, uint32_t (&D)[MAXG]) {
  uint32_t carry = 0;
#pragma unroll
  for (int g = MAXG - 1; g >= 0; --g) {
    const uint32_t d = D[g] + dD[g] + carry;
    carry = d >= R[g] ? 1u : 0u;
    D[g] = carry ? d - R[g] : d;
  }
}

// ---------------------------------------------------------------- top-k
struct TopkShared {
  surr_record* lists;  // [2][k]
  surr_record* cand;   // [num epilogue warps][CAND_CAP]
  volatile uint32_t* misc;  // [0] lock, [1] cur, [2] thr_key, [3..4] thr_idx, [5] valid entries of the list,
                            // [8 + b] candidates left in buffer b at the end (topk_post)
};

__device__ __forceinline__ uint32_t lower_bound_recs(const surr_record* a, uint32_t n, uint32_t key, uint64_t idx) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    surr_record r = a[mid];
    if (rec_less(r.key, r.idx, key, idx)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t upper_bound_recs_fwd(const surr_record* a, uint32_t n, uint32_t key, uint64_t idx) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const surr_record r = a[mid];
    if (!rec_less(key, idx, r.key, r.idx)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Merge the warp's cnt (<= CAND_CAP) candidates into the CTA list (caller
// holds the lock).  misc[5] = nv, the list's valid prefix (L[nv..k) are
// sentinels, candidates never are), so the work is O(nv + cnt), not O(k),
// while the list fills.  Every candidate's insertion point ub_j = #{L < c_j}
// comes from one binary search over L; the candidates are written, then the
// ub_j (ascending) replace them in the warp's buffer as a compact word array
// and each lane walks its L elements' shifts #{j : ub_j <= i} with a pointer.
__device__ void warp_merge(TopkShared& ts, surr_record* cand, uint32_t cnt, uint32_t k, uint32_t lane) {
  // 1. sort candidates by rank (all keys distinct: idx unique)
  surr_record c0, c1;
  uint32_t r0 = 0, r1 = 0;
  bool h0 = lane < cnt, h1 = lane + 32 < cnt;
  if (h0) c0 = cand[lane];
  if (h1) c1 = cand[lane + 32];
  for (uint32_t j = 0; j < cnt; ++j) {
    surr_record o = cand[j];
    if (h0 && rec_less(o.key, o.idx, c0.key, c0.idx)) ++r0;
    if (h1 && rec_less(o.key, o.idx, c1.key, c1.idx)) ++r1;
  }
  // 2. insertion points in the valid prefix of L
  const uint32_t cur = ts.misc[1];
  const uint32_t nv = ts.misc[5];
  surr_record* L = ts.lists + (size_t)cur * k;
  surr_record* O = ts.lists + (size_t)(cur ^ 1u) * k;
  const uint32_t u0 = h0 ? upper_bound_recs_fwd(L, nv, c0.key, c0.idx) : 0u;
  const uint32_t u1 = h1 ? upper_bound_recs_fwd(L, nv, c1.key, c1.idx) : 0u;
  if (nv == 0) {  // first merge: the second buffer's tail becomes sentinels once
    for (uint32_t i = cnt + lane; i < k; i += 32) { O[i].idx = IDX_SENT; O[i].key = KEY_SENT; O[i].pad = 0; }
  }
  // 3. candidates to their final places (rank + insertion point)
  if (h0 && r0 + u0 < k) { c0.pad = 0; O[r0 + u0] = c0; }
  if (h1 && r1 + u1 < k) { c1.pad = 0; O[r1 + u1] = c1; }
  __syncwarp();
  uint32_t* ub = reinterpret_cast<uint32_t*>(cand);  // the candidates are placed: reuse the buffer
  if (h0) ub[r0] = u0;
  if (h1) ub[r1] = u1;
  __syncwarp();
  // 4. L's valid elements shift by the number of candidates inserted before them
  uint32_t jp = 0;
  for (uint32_t i = lane; i < nv; i += 32) {
    while (jp < cnt && ub[jp] <= i) ++jp;
    if (i + jp < k) O[i + jp] = L[i];
  }
  __syncwarp();
  if (lane == 0) {
    surr_record last = O[k - 1];
    ts.misc[1] = cur ^ 1u;
    ts.misc[5] = min(nv + cnt, k);
    ts.misc[3] = (uint32_t)last.idx;
    ts.misc[4] = (uint32_t)(last.idx >> 32);
    ts.misc[2] = last.key;
  }
  __syncwarp();
}

// End of the sweep (a8): each warp posts how many candidates its buffer still
// holds (misc[8 + b] for buffer b, zero-initialised), and after the CTA barrier
// warp 0 merges every posted buffer into the list in buffer order, with no lock
// hand-offs (16 warps contending for the lock at the end cost ~60 us per sweep,
// measured).  The result is the same exact (key, idx) top-k for any order.
constexpr uint32_t TOPK_MAX_BUFS = 16;
__device__ __forceinline__ void topk_post(TopkShared& ts, const surr_record* mycand, uint32_t ncand, uint32_t lane) {
  if (lane == 0) ts.misc[8 + (uint32_t)(mycand - ts.cand) / CAND_CAP] = ncand;
}
// All threads of the CTA, after the barrier that follows every warp's
// topk_post: the candidates left in the buffers are merged into the list in
// one parallel rank merge (each candidate's position = #candidates below it
// + #list entries below it; each list entry's = its index + #candidates below
// it), so the end of a sweep costs one pass instead of one warp_merge per
// buffer in sequence (~2.5 us each; 73-80 % of a one-tile-per-slot sweep's
// time, ncu).  The caller synchronises the CTA before reading the list.
__device__ void topk_drain(TopkShared& ts, uint32_t k, uint32_t /*warp*/, uint32_t /*lane*/) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  // buffer b holds misc[8 + b] candidates (read from shared memory where needed:
  // a register array indexed at run time would live in local memory)
  uint32_t tot = 0;
#pragma unroll
  for (uint32_t b = 0; b < TOPK_MAX_BUFS; ++b) tot += ts.misc[8 + b];
  if (tot == 0) return;  // (uniform)
  const uint32_t cur = ts.misc[1], nv = ts.misc[5];
  const surr_record* L = ts.lists + (size_t)cur * k;
  surr_record* O = ts.lists + (size_t)(cur ^ 1u) * k;
  const uint32_t nout = min(nv + tot, k);
  // #candidates strictly below (key, idx): every thread walks the buffers in the same order (broadcast loads)
  auto below = [&](uint32_t key, uint64_t idx) {
    uint32_t r = 0;
#pragma unroll 1
    for (uint32_t b = 0; b < TOPK_MAX_BUFS; ++b) {
      const surr_record* cb = ts.cand + (size_t)b * CAND_CAP;
      const uint32_t nb = ts.misc[8 + b];
      for (uint32_t j = 0; j < nb; ++j) {
        const surr_record o = cb[j];
        r += rec_less(o.key, o.idx, key, idx) ? 1u : 0u;
      }
    }
    return r;
  };
  for (uint32_t i = nout + t; i < k; i += nt) { O[i].idx = IDX_SENT; O[i].key = KEY_SENT; O[i].pad = 0; }
  for (uint32_t g = t; g < tot; g += nt) {  // candidate g of the flattened buffers
    uint32_t b = 0, j = g;
    for (uint32_t nb = ts.misc[8]; j >= nb; nb = ts.misc[8 + b]) { j -= nb; ++b; }
    surr_record c = ts.cand[(size_t)b * CAND_CAP + j];
    const uint32_t pos = below(c.key, c.idx) + upper_bound_recs_fwd(L, nv, c.key, c.idx);
    c.pad = 0;
    if (pos < k) O[pos] = c;
  }
  for (uint32_t i = t; i < nv; i += nt) {
    const surr_record e = L[i];
    const uint32_t pos = i + below(e.key, e.idx);
    if (pos < k) O[pos] = e;
  }
  __syncthreads();
  if (t == 0) {
    const surr_record last = O[k - 1];
    ts.misc[1] = cur ^ 1u;
    ts.misc[5] = nout;
    ts.misc[3] = (uint32_t)last.idx;
    ts.misc[4] = (uint32_t)(last.idx >> 32);
    ts.misc[2] = last.key;
  }
}

__device__ __forceinline__ void lock_acquire(TopkShared& ts, uint32_t lane) {
  if (lane == 0) {
    while (atomicCAS((uint32_t*)&ts.misc[0], 0u, 1u) != 0u) __nanosleep(32);
    __threadfence_block();
  }
  __syncwarp();
}
__device__ __forceinline__ void lock_release(TopkShared& ts, uint32_t lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    atomicExch((uint32_t*)&ts.misc[0], 0u);
  }
}


// ------------------------------------------------------------------ K2
// Merge `lists` sorted lists of k_in records into the k best (one CTA):
// lists are loaded a chunk at a time (coalesced, all threads), reduced by a
// pairwise tree of rank merges in shared memory, then merged into the result.
// Ties (only sentinels can tie) are broken by list order: elements of the
// left list use count(right < e), of the right list count(left <= f), so the
// output positions are a permutation.
__device__ __forceinline__ uint32_t upper_bound_recs(const surr_record* a, uint32_t n, uint32_t key, uint64_t idx) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const surr_record r = a[mid];
    if (!rec_less(key, idx, r.key, r.idx)) lo = mid + 1; else hi = mid;  // r <= (key, idx)
  }
  return lo;
}

// out[0..min(na+nb, cap)) = first elements of merge(A[0..na), B[0..nb))
__device__ __forceinline__ void rank_merge(const surr_record* A, uint32_t na, const surr_record* B, uint32_t nb,
                                           surr_record* out, uint32_t cap, uint32_t t, uint32_t nt) {
  for (uint32_t i = t; i < na; i += nt) {
    const surr_record e = A[i];
    const uint32_t pp = i + lower_bound_recs(B, nb, e.key, e.idx);
    if (pp < cap) out[pp] = e;
  }
  for (uint32_t i = t; i < nb; i += nt) {
    const surr_record f = B[i];
    const uint32_t pp = i + upper_bound_recs(A, na, f.key, f.idx);
    if (pp < cap) out[pp] = f;
  }
}

// The merge body, run by every thread of one CTA over `sm` (shared memory of
// (2 k + 2 chunk max(k_in, k)) records).  CG: read the lists with ld.global.cg
// (written by other CTAs of the same launch).
template <bool CG>
__device__ void merge_lists(const surr_record* __restrict__ in, uint32_t lists, uint32_t k_in, uint32_t k,
                            uint32_t chunk, uint64_t* out_idx, float* out_t, surr_record* out_recs, uint8_t* sm) {
  // list slots are S = max(k_in, k) records apart, so a merged list (up to k
  // records) never overruns its neighbour when k > k_in
  const uint32_t S = max(k_in, k);
  surr_record* T = reinterpret_cast<surr_record*>(sm);  // [k] result so far
  surr_record* T2 = T + k;                              // [k]
  surr_record* X = T2 + k;                              // [chunk * S]
  surr_record* Y = X + (size_t)chunk * S;               // [chunk * S]
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  for (uint32_t i = t; i < k; i += nt) { T[i].idx = IDX_SENT; T[i].key = KEY_SENT; T[i].pad = 0; }
  for (uint32_t c0 = 0; c0 < lists; c0 += chunk) {
    const uint32_t m = min(chunk, lists - c0);
    const uint4* src = reinterpret_cast<const uint4*>(in + (size_t)c0 * k_in);
    auto ld = [&](uint32_t i) { return CG ? __ldcg(src + i) : src[i]; };
    if (S == k_in) {
      for (uint32_t i = t; i < m * k_in; i += nt) reinterpret_cast<uint4*>(X)[i] = ld(i);
    } else {
      for (uint32_t i = t; i < m * k_in; i += nt) reinterpret_cast<uint4*>(X)[(i / k_in) * S + i % k_in] = ld(i);
    }
    __syncthreads();
    // pairwise tree: nl lists of length len (stride S) -> ceil(nl/2) lists of length min(2 len, k)
    uint32_t nl = m, len = k_in;
    const uint32_t st = S;
    surr_record *cur = X, *nxt = Y;
    while (nl > 1) {
      const uint32_t nlen = min(2 * len, k);
      const uint32_t pairs = nl / 2;
      // threads split across pairs
      const uint32_t tpp = max(1u, nt / pairs);
      const uint32_t pr = t / tpp, tt = t % tpp;
      for (uint32_t pi = pr; pi < pairs; pi += max(1u, nt / tpp)) {
        rank_merge(cur + (size_t)(2 * pi) * st, len, cur + (size_t)(2 * pi + 1) * st, len, nxt + (size_t)pi * st,
                   nlen, tt, tpp);
      }
      if (nl & 1) {
        for (uint32_t i = t; i < len; i += nt) nxt[(size_t)pairs * st + i] = cur[(size_t)(nl - 1) * st + i];
        for (uint32_t i = len + t; i < nlen; i += nt) {
          nxt[(size_t)pairs * st + i].idx = IDX_SENT; nxt[(size_t)pairs * st + i].key = KEY_SENT;
          nxt[(size_t)pairs * st + i].pad = 0;
        }
      }
      __syncthreads();
      surr_record* tmp = cur; cur = nxt; nxt = tmp;
      nl = (nl + 1) / 2;
      len = nlen;
    }
    // merge the chunk's best (cur[0..len)) into T
    rank_merge(T, k, cur, min(len, k), T2, k, t, nt);
    __syncthreads();
    surr_record* tmp = T; T = T2; T2 = tmp;
  }
  for (uint32_t i = t; i < k; i += nt) {
    const surr_record e = T[i];
    if (out_idx) out_idx[i] = e.idx;
    if (out_t) out_t[i] = key2f(e.key);
    if (out_recs) out_recs[i] = e;
  }
}

__global__ void __launch_bounds__(1024, 1)
    merge_kernel(const surr_record* __restrict__ in, uint32_t lists, uint32_t k_in, uint32_t k, uint32_t chunk,
                 uint64_t* out_idx, float* out_t, surr_record* out_recs) {
  extern __shared__ __align__(16) uint8_t sm[];
  merge_lists<false>(in, lists, k_in, k, chunk, out_idx, out_t, out_recs, sm);
}

// a9 fused into K1 (MODE_TOPK, p.done_ctr set) as a binary tree of CTAs: every
// CTA has written its k records to p.recs[blockIdx.x k ..]; at level l the
// node j covers CTAs [j 2^l, (j + 1) 2^l) and its list sits in the slot of its
// leftmost CTA (j 2^l).  Of the two children of a node, the one that finishes
// second (device-scope ticket per node, re-armed by that CTA) merges both
// lists (staged in its shared memory) into the left child's slot and climbs;
// the other one exits.  A node without a sibling (odd count) climbs without a
// merge.  The CTA that completes the root writes the outputs.  The critical
// path is log2(grid) two-list merges (~8 at 148 CTAs) instead of one CTA
// merging every list (the chunked K2 loop: ~1 ms at k = 1024, measured).
// Ties (only sentinels can tie) keep list order, so the result is the unique
// (key, idx) top-k.  Called by every thread of the CTA after the teardown.
constexpr uint32_t TREE_NODES_PER_LEVEL = 256;  // ticket array: levels x 256 counters (grid <= 256)
__device__ __forceinline__ void grid_merge_tail(const KParams& p, int mode, uint8_t* sm) {
  if (mode != MODE_TOPK || p.done_ctr == nullptr) return;
  const uint32_t k = p.k, t = threadIdx.x, nt = blockDim.x;
  surr_record* A = reinterpret_cast<surr_record*>(sm);
  surr_record* B = A + k;
  surr_record* O = B + k;
  uint32_t node = blockIdx.x, nodes = gridDim.x, l = 0;
  bool merged = false;  // O holds this CTA's latest merge result
  for (; nodes > 1; ++l) {
    if ((node ^ 1u) < nodes) {
      __syncthreads();  // this CTA's list (or merge result) is written
      int second = 0;
      if (t == 0) {
        uint32_t* tk = p.done_ctr + l * TREE_NODES_PER_LEVEL + (node >> 1);
        __threadfence();  // release: the list before the ticket
        second = atomicAdd(tk, 1u) == 1u;
        if (second) {
          __threadfence();  // acquire: the sibling's list
          *tk = 0u;         // re-armed for the next launch (nobody else touches it in this one)
        }
      }
      if (!__syncthreads_or(second)) return;  // the sibling merges
      const surr_record* L = p.recs + (size_t)((node & ~1u) << l) * k;
      const surr_record* R = p.recs + (size_t)((node | 1u) << l) * k;
      for (uint32_t i = t; i < k; i += nt) {
        reinterpret_cast<uint4*>(A)[i] = __ldcg(reinterpret_cast<const uint4*>(L) + i);
        reinterpret_cast<uint4*>(B)[i] = __ldcg(reinterpret_cast<const uint4*>(R) + i);
      }
      __syncthreads();
      rank_merge(A, k, B, k, O, k, t, nt);
      __syncthreads();
      merged = true;
      if (nodes > 2) {  // not the root: the result goes to the parent's slot (= the left child's)
        surr_record* P = p.recs + (size_t)((node & ~1u) << l) * k;
        for (uint32_t i = t; i < k; i += nt) reinterpret_cast<uint4*>(P)[i] = reinterpret_cast<const uint4*>(O)[i];
      }
    }
    node >>= 1;
    nodes = (nodes + 1) >> 1;
  }
  // the root: this CTA's merge result (or, grid of one, its own list)
  __syncthreads();
  const surr_record* src = merged ? O : p.recs + (size_t)blockIdx.x * k;
  for (uint32_t i = t; i < k; i += nt) {
    surr_record e;
    if (merged) {
      e = src[i];
    } else {
      const uint4 u = __ldcg(reinterpret_cast<const uint4*>(src) + i);
      e = *reinterpret_cast<const surr_record*>(&u);
    }
    if (p.out_idx) p.out_idx[i] = e.idx;
    if (p.out_t) p.out_t[i] = key2f(e.key);
    if (p.out_recs) p.out_recs[i] = e;
  }
}

// A0 operand of one row: bf16 / fp16 -> 8 packed columns; 3xFP16 -> 8 hi + 8 lo
// packed columns; tf32 -> 16 hi + 16 lo slots.
struct A0Regs {
  uint32_t hi[K0], lo[K0];
};

// a3: one table lookup per group (pre-normalised, pre-rounded slot pairs)
template <int PREC>
__device__ __forceinline__ void make_a0_sweep(const KParams& p, const uint8_t* slut, const uint32_t (&D)[MAXG],
                                              A0Regs& a) {
#pragma unroll
  for (int g = 0; g < MAXG; ++g) {
    if (is16(PREC)) {
      a.hi[g] = reinterpret_cast<const uint32_t*>(slut)[p.lut_off[g] + D[g]];
    } else if (PREC == PREC_FP32H) {  // 8-byte entry: fp16 hi pair, fp16 lo pair
      const uint2 e = reinterpret_cast<const uint2*>(slut)[p.lut_off[g] + D[g]];
      a.hi[g] = e.x;
      a.lo[g] = e.y;
    } else {
      const uint4 e = reinterpret_cast<const uint4*>(slut)[p.lut_off[g] + D[g]];
      a.hi[2 * g] = e.x; a.hi[2 * g + 1] = e.y; a.lo[2 * g] = e.z; a.lo[2 * g + 1] = e.w;
    }
  }
}

// 4-slot groups (bf16): one 8-byte table entry = two packed A0 columns
__device__ __forceinline__ void make_a0_sweep4(const KParams& p, const uint8_t* slut, const uint32_t (&D)[MAXG],
                                               A0Regs& a) {
#pragma unroll
  for (int g = 0; g < K0 / 4; ++g) {
    const uint2 e = reinterpret_cast<const uint2*>(slut)[p.lut_off[g] + D[g]];
    a.hi[2 * g] = e.x;
    a.hi[2 * g + 1] = e.y;
  }
}

// MODE_A0 (parity hook): the layer-1 operand row the sweep built for config I
// (every a0_stride-th config of the range, so whole-space launches can be sampled),
// exactly as it is stored for the UMMA (8 packed hi columns, 8 lo columns; LO =
// false: 16-bit kernels, whose lo words are written as 0)
template <bool LO>
__device__ __forceinline__ void a0_dump(const KParams& p, int mode, const A0Regs& a, uint64_t I) {
  if (mode == MODE_A0 && I < p.end) {
    const uint64_t off = I - p.begin, q = off / p.a0_stride;  // every a0_stride-th config
    if (q * p.a0_stride != off) return;
    uint4* o = reinterpret_cast<uint4*>(p.a0_dump + q * 16);
    o[0] = make_uint4(a.hi[0], a.hi[1], a.hi[2], a.hi[3]);
    o[1] = make_uint4(a.hi[4], a.hi[5], a.hi[6], a.hi[7]);
    o[2] = LO ? make_uint4(a.lo[0], a.lo[1], a.lo[2], a.lo[3]) : make_uint4(0u, 0u, 0u, 0u);
    o[3] = LO ? make_uint4(a.lo[4], a.lo[5], a.lo[6], a.lo[7]) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// explicit-batch rows: z_j = (x_j - shift_j) * (1 / scale_j) in double (the host
// table divides; the two agree to 1 ulp of double before the fp32 rounding),
// slot P = 1 (bias), rest 0.  Column pairs are loaded (8-byte loads when P is
// even) and converted one at a time to keep the live register set small.
// PC >= 0: the parameter count as a compile-time constant (the paper's 14: no
// per-slot compares); PC < 0: runtime p.P
template <int PREC, bool SMEM, int PC>
__device__ __forceinline__ void make_a0_row_n(const KParams& p, const float* xr, A0Regs& a) {
  const int P = PC >= 0 ? PC : (int)p.P;
  const bool even = (P & 1) == 0;
  // global rows: read-only path; staged rows: plain shared-memory loads
  auto ld2 = [&](int j) { return SMEM ? *reinterpret_cast<const float2*>(xr + j) : __ldg(reinterpret_cast<const float2*>(xr + j)); };
  auto ld1 = [&](int j) { return SMEM ? xr[j] : __ldg(xr + j); };
#pragma unroll
  for (int j = 0; j < K0; j += 2) {
    float x0 = 0.0f, x1 = 0.0f;
    if (j + 1 < P && even) {
      const float2 v = ld2(j);
      x0 = v.x;
      x1 = v.y;
    } else {
      if (j < P) x0 = ld1(j);
      if (j + 1 < P) x1 = ld1(j + 1);
    }
    float z0 = 0.0f, z1 = 0.0f;
    if (j < P) z0 = fmaf(x0, p.zinv[j], p.zc[j]);
    else if (j == P) z0 = 1.0f;
    if (j + 1 < P) z1 = fmaf(x1, p.zinv[j + 1], p.zc[j + 1]);
    else if (j + 1 == P) z1 = 1.0f;
    if (is16(PREC)) {
      a.hi[j / 2] = pk16<PREC>(z0, z1);
    } else if (PREC == PREC_FP32H) {  // fp16 hi + fp16(z - hi) lo
      a.hi[j / 2] = f16x2(z0, z1);
      float h0, h1;
      f16x2_to_f32(a.hi[j / 2], h0, h1);
      a.lo[j / 2] = f16x2(z0 - h0, z1 - h1);
    } else {
      a.hi[j] = to_tf32(z0);
      a.lo[j] = __float_as_uint(z0 - __uint_as_float(a.hi[j]));  // exact; the UMMA truncates it to tf32
      a.hi[j + 1] = to_tf32(z1);
      a.lo[j + 1] = __float_as_uint(z1 - __uint_as_float(a.hi[j + 1]));
    }
  }
}
template <int PREC, bool SMEM = false>
__device__ __forceinline__ void make_a0_row(const KParams& p, const float* xr, A0Regs& a) {
  if (p.P == 14) make_a0_row_n<PREC, SMEM, 14>(p, xr, a);
  else make_a0_row_n<PREC, SMEM, -1>(p, xr, a);
}
template <int PREC>
__device__ __forceinline__ void make_a0_predict(const KParams& p, uint64_t r, A0Regs& a) {
  make_a0_row<PREC>(p, p.x + r * p.P, a);
}

template <int PREC, int H>
__global__ void __launch_bounds__(Cfg<PREC, H>::THREADS, 1)
    sweep_kernel(const __grid_constant__ KParams p, int mode) {
  using C = Cfg<PREC, H>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_misc);  // [0] load, [1..2] a, [3..4] d
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.smem_misc + 64);
  TopkShared ts;
  ts.lists = reinterpret_cast<surr_record*>(smem + p.smem_lists);
  ts.cand = reinterpret_cast<surr_record*>(smem + p.smem_cand);
  ts.misc = reinterpret_cast<volatile uint32_t*>(smem + p.smem_misc + 128);

  // ---- setup
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < C::NSLOT; ++s) {
        mbar_init(&bars[1 + s], 4);  // one arrive per epilogue warp of the slot
        mbar_init(&bars[3 + s], 1);  // tcgen05.commit
      }
      fence_mbar_init();
      fence_proxy_async_smem();
      // weights (+ value table) -> smem through the bulk-copy engine, one mbarrier
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
  if (C::BIAS_MMA && warp >= 4 && warp < 8) {
    // constant ones block (A operand of the bias K step): slot 0 = 1, rest 0
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0u;
    ones[0] = is16(PREC) ? one16<PREC>() : 0x3F800000u;
    tmem_st8(tmem_base + (((warp & 3u) * 32u) << 16) + C::ONES_COL, ones);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ================= UMMA issuer (warp 0, converged) =================
    // Round-robin over slots, layer by layer; waits are blocking (HW-suspending)
    // try_waits.  The whole warp runs the loop so descriptor arithmetic stays
    // warp-uniform; one elected lane issues each layer's fully unrolled UMMA
    // chain (issue cost ~ a few cycles per UMMA instead of ~40 in divergent code).
    mbar_wait(&bars[0], 0);  // weights resident
    uint32_t ntile[C::NSLOT], ph[C::NSLOT];
    uint32_t rounds = 0;
#pragma unroll
    for (int s = 0; s < C::NSLOT; ++s) {
      const uint64_t t0 = (uint64_t)blockIdx.x * C::NSLOT + s;
      ntile[s] = t0 < p.num_tiles ? (uint32_t)((p.num_tiles - t0 - 1) / p.dTiles + 1) : 0u;
      ph[s] = 0;
      rounds = max(rounds, ntile[s]);
    }
    const uint32_t sb = smem_u32(smem);
    const uint32_t ones = tmem_base + C::ONES_COL;
    const uint64_t d_b1 = make_bdesc(sb + p.off_b1, p.sbo_b1);
    const uint64_t d_b1lo = make_bdesc(sb + p.off_b1lo, p.sbo_b1);
    const uint32_t idesc = p.idesc;
    for (uint32_t j = 0; j < rounds; ++j) {
      for (uint32_t l = 0; l < p.NL; ++l) {
        const uint64_t d_bh = make_bdesc(sb + p.off_bh + (l ? l - 1 : 0) * p.stride_bh, p.sbo_bh);
        const uint64_t d_bhlo = make_bdesc(sb + p.off_bh + (l ? l - 1 : 0) * p.stride_bh + p.lo_delta_h, p.sbo_bh);
#pragma unroll
        for (int s = 0; s < C::NSLOT; ++s) {
          if (j >= ntile[s]) continue;
          mbar_wait(&bars[1 + s], ph[s]);
          ph[s] ^= 1u;
          tc_fence_after();
          const uint32_t d = tmem_base + s * C::SLOT_COLS;
          const uint32_t a = d + H;
          if (elect_one()) {
            if (l == 0) {
              // K0 = 16: one bf16 step, or two tf32 steps x 3 passes
#pragma unroll
              for (int kk = 0; kk < K0 / C::KSTEP; ++kk) {
                if (is16(PREC)) {
                  umma_f16_ts(d, a + kk * 8, d_b1 + kk * 16, idesc, kk > 0);
                } else {
                  umma_tf32_ts(d, a + kk * 8, d_b1 + kk * 16, idesc, kk > 0);
                  umma_tf32_ts(d, a + kk * 8, d_b1lo + kk * 16, idesc, 1u);
                  umma_tf32_ts(d, a + C::A0_LO + kk * 8, d_b1 + kk * 16, idesc, 1u);
                }
              }
            } else {
#pragma unroll
              for (int kk = 0; kk < H / C::KSTEP; ++kk) {
                if (is16(PREC)) {
                  umma_f16_ts(d, a + kk * 8, d_bh + kk * 16, idesc, kk > 0);
                } else {
                  umma_tf32_ts(d, a + kk * 8, d_bh + kk * 16, idesc, kk > 0);
                  if (C::PASSES_H == 3) {
                    umma_tf32_ts(d, a + kk * 8, d_bhlo + kk * 16, idesc, 1u);
                    umma_tf32_ts(d, a + H + kk * 8, d_bh + kk * 16, idesc, 1u);
                  }
                }
              }
              if (C::BIAS_MMA) {  // D += ones * [b; 0] (the B image carries one extra K block)
                constexpr int kb = H / C::KSTEP;
                if (is16(PREC)) {
                  umma_f16_ts(d, ones, d_bh + kb * 16, idesc, 1u);
                } else {
                  umma_tf32_ts(d, ones, d_bh + kb * 16, idesc, 1u);
                  if (C::PASSES_H == 3) umma_tf32_ts(d, ones, d_bhlo + kb * 16, idesc, 1u);
                }
              }
            }
            umma_commit(&bars[3 + s]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    // ================= slot warpgroups: rows, epilogues, top-k =================
    const uint32_t s = (warp >> 2) - 1;
    const uint32_t wq = warp & 3u;
    const uint32_t row = wq * 32u + lane;
    const uint32_t tl = (wq * 32u) << 16;  // TMEM lane offset of this warp
    const uint32_t dcol = tmem_base + tl + s * C::SLOT_COLS;
    const uint32_t acol = dcol + H;
    const uint8_t* slut = smem + p.smem_lut;
    surr_record* mycand = ts.cand + (size_t)(warp - 4) * CAND_CAP;
    uint32_t ncand = 0;

    uint64_t tile = (uint64_t)blockIdx.x * C::NSLOT + s;
    uint64_t I = p.begin + tile * TILE_M + row;
    const uint64_t dI = (uint64_t)p.dTiles * TILE_M;
    uint32_t D[MAXG];
    if (mode != MODE_PREDICT) init_digits(p.R, I, D);
    uint32_t phd = 0;
    mbar_wait(&bars[0], 0);  // table / weights resident

    // software pipeline: the A0 operand of the NEXT tile is built while the
    // last UMMA layer of the current tile runs
    A0Regs a0;
    if (tile < p.num_tiles) {
      if (mode == MODE_PREDICT) make_a0_predict<PREC>(p, I < p.end ? I : p.begin, a0);
      else make_a0_sweep<PREC>(p, slut, D, a0);
    }
    for (; tile < p.num_tiles; tile += p.dTiles) {
      const bool valid = I < p.end;
    const float accp = ens_prefetch(p, valid, I);
      // ---------------- a2 + a3: A0 operand -> TMEM
      if (is16(PREC)) {
        tmem_st8(acol, a0.hi);
      } else {
        tmem_st16(acol, a0.hi);
        tmem_st16(acol + C::A0_LO, a0.lo);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[1 + s]);

      const uint64_t In = I + dI;
      const bool has_next = tile + p.dTiles < p.num_tiles;

      // ---------------- layers
      float t = 0.0f;
      for (uint32_t l = 0; l < p.NL; ++l) {
        if (l + 1 == p.NL && has_next) {
          if (mode == MODE_PREDICT) {
            make_a0_predict<PREC>(p, In < p.end ? In : p.begin, a0);
          } else {
            odometer_step(p.R, p.dD, D);
            make_a0_sweep<PREC>(p, slut, D, a0);
          }
        }
        mbar_wait(&bars[3 + s], phd);
        phd ^= 1u;
        tc_fence_after();
        if (l + 1 < p.NL) {
          // a5: hidden epilogue -> next A operand (two 32-column chunks per TMEM wait)
#pragma unroll
          for (int c = 0; c < H / 32; c += 2) {
            uint32_t v[2][32];
            tmem_ld32(dcol + c * 32, v[0]);
            if (H / 32 > 1) tmem_ld32(dcol + (c + 1) * 32, v[1]);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u == 1 && H / 32 == 1) break;
              const int cc = c + u;
              if (!C::BIAS_MMA && l >= 1) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  v[u][j] = __float_as_uint(__uint_as_float(v[u][j]) + p.hbias[(l - 1) & 1][cc * 32 + j]);
              }
              if (is16(PREC)) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  pk[j] = relu_pk16<PREC>(__uint_as_float(v[u][2 * j]), __uint_as_float(v[u][2 * j + 1]));
                tmem_st16(acol + cc * 16, pk);
              } else {
                uint32_t hv[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const float x = fmaxf(__uint_as_float(v[u][j]), 0.0f);
                  hv[j] = to_tf32(x);
                  if (PREC == PREC_FP32) v[u][j] = __float_as_uint(x - __uint_as_float(hv[j]));
                }
                tmem_st32(acol + cc * 32, hv);
                if (PREC == PREC_FP32) tmem_st32(acol + H + cc * 32, v[u]);
              }
            }
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[1 + s]);
        } else {
          // a7: FP32 final layer, packed FFMA2 over column pairs, 4 accumulator pairs;
          // ReLU threshold 0 when the bias is in D, else relu(x + b) = max(x, -b) + b
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int c = 0; c < H / 32; c += 2) {
            uint32_t v[2][32];
            tmem_ld32(dcol + c * 32, v[0]);
            if (H / 32 > 1) tmem_ld32(dcol + (c + 1) * 32, v[1]);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u == 1 && H / 32 == 1) break;
              const int cc = c + u;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const uint64_t w2 = pack2(p.fin_w[cc * 32 + j], p.fin_w[cc * 32 + j + 1]);
                if (C::BIAS_MMA) {
                  // w relu(x) = (w/2) x + (w/2) |x|  (fin_w holds w/2; |x| is a free FFMA2 operand modifier)
                  const uint64_t x2 = pack2(__uint_as_float(v[u][j]), __uint_as_float(v[u][j + 1]));
                  const uint64_t a2 = pack2(fabsf(__uint_as_float(v[u][j])), fabsf(__uint_as_float(v[u][j + 1])));
                  acc[(j >> 1) & 1] = ffma2(w2, x2, acc[(j >> 1) & 1]);
                  acc[2 + ((j >> 1) & 1)] = ffma2(w2, a2, acc[2 + ((j >> 1) & 1)]);
                } else {
                  const float x0 = fmaxf(__uint_as_float(v[u][j]), p.fin_nb[cc * 32 + j]);
                  const float x1 = fmaxf(__uint_as_float(v[u][j + 1]), p.fin_nb[cc * 32 + j + 1]);
                  acc[(j >> 1) & 3] = ffma2(w2, pack2(x0, x1), acc[(j >> 1) & 3]);
                }
              }
            }
          }
          float a8[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) unpack2(acc[j], a8[2 * j], a8[2 * j + 1]);
          t = (((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]))) + p.c_out;
        }
      }

      // ---------------- outputs
      if (!ens_stage(p, valid, I, t, accp)) {
      } else if (mode == MODE_TOPK) {
        const uint32_t key = f2key(t);
        // conservative filter on the key alone (a stale read only admits extra
        // candidates; the merge keeps the exact (key, idx) top-k)
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
      I = In;
    }
    if (mode == MODE_TOPK) topk_post(ts, mycand, ncand, lane);
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
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  grid_merge_tail(p, mode, smem);
}

// ------------------------------------------------------------ decode hook
// The kernels' decoder on arbitrary ranges: each thread initialises its digits
// once and then advances by the grid stride with the same odometer.
struct DecodeParams {
  uint32_t R[MAXG], dD[MAXG];   // group radices, digits of the grid stride
  uint32_t radix[32];
  uint32_t P, spg;              // parameters; parameter slots per group
  uint64_t first, n;
  uint8_t* out;
};

__global__ void decode_kernel(const __grid_constant__ DecodeParams p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t D[MAXG];
  init_digits(p.R, p.first + i, D);
  for (; i < p.n; i += stride) {
    for (uint32_t g = 0; p.spg * g < p.P; ++g) {
      uint32_t rem = D[g];
      for (int q = (int)p.spg - 1; q >= 0; --q) {
        const uint32_t slot = p.spg * g + q;
        const uint32_t r = slot < p.P ? p.radix[slot] : 1u;
        if (slot < p.P) p.out[i * p.P + slot] = (uint8_t)(rem % r);
        rem /= r;
      }
    }
    odometer_step(p.R, p.dD, D);
  }
}

// ------------------------------------------------------------ UMMA self-test
// One 128 x N x K GEMM: A rows staged to TMEM with tcgen05.st, B bulk-copied
// to shared memory, D read back with tcgen05.ld.  Test infrastructure for the
// descriptor / layout encodings the sweep kernel relies on.
__global__ void __launch_bounds__(128, 1)
    umma_selftest_kernel(const uint32_t* A, uint32_t K, uint32_t acols, const uint8_t* B, uint32_t bbytes,
                         float* Dout, uint32_t N, int bf, uint32_t idesc, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ((bbytes + 127u) / 128u) * 128u);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_mbar_init();
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[0], bbytes);
      for (uint32_t off = 0; off < bbytes; off += 32768u)
        bulk_g2s(smem + off, B + off, min(32768u, bbytes - off), &bars[0]);
    }
    __syncwarp();
    tmem_alloc<512>(tslot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = *tslot;
  const uint32_t row = threadIdx.x;
  const uint32_t tl = (warp * 32u) << 16;
  for (uint32_t c = 0; c < acols; c += 8) {
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = A[(size_t)row * K + c + j];
    tmem_st8(base + tl + N + c, v);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint32_t steps = bf ? K / 16 : K / 8;
    for (uint32_t kk = 0; kk < steps; ++kk) {
      const uint64_t d = make_bdesc(smem_u32(smem) + kk * 256u, sbo);
      if (bf) umma_f16_ts(base, base + N + kk * 8u, d, idesc, kk > 0);
      else umma_tf32_ts(base, base + N + kk * 8u, d, idesc, kk > 0);
    }
    umma_commit(&bars[1]);
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  for (uint32_t c = 0; c < N; c += 32) {
    uint32_t v[32];
    tmem_ld32(base + tl + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) Dout[(size_t)row * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(base, 512);
  }
}

}  // namespace surr
