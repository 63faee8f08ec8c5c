// GPU-side training of the FCNN surrogate: the paper's
// scikit-learn MLPRegressor recipe (Table "Hyperparameter" P:212-235;
// the same algorithm oracle/mlp.py restates in float64) in FP32 on the GPU.
//
// Per minibatch of B <= 200 rows (the last one short), for F-H-H-1 nets:
//   h1 = relu(X W1 + b1), h2 = relu(h1 W2 + b2), yhat = h2 W3 + b3
//   loss = 1/2 mean (yhat - y)^2 + alpha / (2B) sum ||W||_F^2      (biases excluded)
//   d3 = yhat - y; gW3 = (h2^T d3 + alpha W3)/B; gb3 = mean d3
//   d2 = d3 W3^T . [h2 > 0]; gW2 = (h1^T d2 + alpha W2)/B; gb2 = mean d2
//   d1 = d2 W2^T . [h1 > 0]; gW1 = (X^T d1 + alpha W1)/B; gb1 = mean d1
//   Adam (sklearn form): m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2,
//   lr_t = lr0 sqrt(1 - b2^t) / (1 - b1^t), p -= lr_t m / (sqrt(v) + eps)
// Epoch loss = sample-weighted mean of the batch losses; training stops after
// more than n_iter_no_change epochs without improving the best loss by tol.
//
// B200 mapping: ONE launch for the whole fit.  Each ensemble member (SURVEY
// G15: members differ in initialisation and epoch orders) is a thread-block
// cluster of C = H / 16 CTAs (8 at H = 128) resident for every epoch, so an
// 8-member ensemble occupies 64 SMs at once.  CTA c owns the 16 hidden units
// [16c, 16c + 16) of both hidden layers: its columns of W1, W2, W3 and their
// Adam state, and computes those units' activations and deltas for the whole
// batch.  Layers meet through distributed shared memory: each CTA gathers the
// other CTAs' 16-unit slices of h1 (forward) and of d2 (backward) into its own
// full-width buffer, the output is a cluster reduction of per-CTA partial dot
// products, and the updated W2 columns are written into every CTA's full W2
// copy (d1 = d2 W2^T reads W2 rows).  Five cluster barriers per step; global
// memory only for the batch rows and the W2 Adam moments.  Activations are
// stored unit-major (A^T[k][r]) so every inner loop is 16-byte shared-memory
// loads of 4 consecutive rows; W2 rows are padded by 4 floats against bank
// conflicts.  FP32 FMA throughout: a step is ~10 MFLOP, latency-bound, not a
// contraction worth splitting into 3xFP16 tensor-core passes.
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

namespace surr {

namespace cg = cooperative_groups;

constexpr int TR_BMAX = 200;  // batch rows held in shared memory (the paper's batch size)
constexpr int TR_FMAX = 20;   // input features (14 parameters + device features)
constexpr int TR_CPC = 16;    // hidden units per CTA
constexpr int TR_THREADS = 256;

struct TrainParams {
  const float* X;         // [n][F] standardised inputs
  const float* y;         // [n] standardised targets
  const uint32_t* perms;  // [E][max_epochs][n] epoch orders (null: identity order)
  uint32_t n, F, B, E;    // rows, features, batch size, ensemble members (clusters)
  uint32_t max_epochs, n_iter_no_change;
  float alpha, beta1, beta2, lr0, eps;
  double tol;
  // member e's parameters start at params + e * pstride: W1 [F][H], b1 [H],
  // W2 [H][H], b2 [H], W3 [H], b3 [1] (fp32, row-major fan_in x fan_out);
  // read as the initial values, overwritten with the trained ones
  float* params;
  uint32_t pstride, oW1, ob1, oW2, ob2, oW3, ob3;
  float* mv;              // Adam moments of the W2 columns: [E][C][2][H][16]
  double* loss_hist;      // [E][max_epochs]
  uint32_t* result;       // [E][3]: epochs run, stop reason (0 max_epochs, 1 tol), Adam steps
  unsigned long long* prof;  // development: per-phase clock64 sums of CTA 0 thread 0 (null: off)
};

template <int H>
struct TrainSmem {
  static constexpr int C = H / TR_CPC;
  static constexpr int WS = H + 4;  // padded W2 row stride (floats)
  float W2[H * WS];               // full copy, row-major [k][n]
  float AT[H * TR_BMAX];          // h1^T (forward), then d2^T (backward): [unit][row]
  float h1T[TR_CPC * TR_BMAX];    // own h1 units, then d1 in place
  float h2T[TR_CPC * TR_BMAX];    // own h2 units, then d2 in place
  float XT[TR_FMAX * TR_BMAX];    // batch inputs, [feature][row]
  float y[TR_BMAX];
  float ypart[TR_BMAX];           // own partial of yhat (read by every CTA)
  float d3[TR_BMAX];              // output deltas; before them, the batch's row indices
  float gW2[H * TR_CPC];          // gradient of the own W2 columns, [k][j]
  float W1o[TR_FMAX * TR_CPC], gW1[TR_FMAX * TR_CPC], mW1[TR_FMAX * TR_CPC], vW1[TR_FMAX * TR_CPC];
  float b1o[TR_CPC], b2o[TR_CPC], W3o[TR_CPC], gb1[TR_CPC], gb2[TR_CPC], gW3[TR_CPC];
  float mb1[TR_CPC], vb1[TR_CPC], mb2[TR_CPC], vb2[TR_CPC], mW3[TR_CPC], vW3[TR_CPC];
  float wsq;                      // own sum of squared weights (read by every CTA)
  float red[TR_THREADS / 32];
  float b3, mb3, vb3, gb3;
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < TR_THREADS / 32; ++i) s += red[i];
  return s;
}

__device__ __forceinline__ void adam(float& p, float& m, float& v, float g, float b1, float b2, float lr_t, float eps) {
  m = b1 * m + (1.0f - b1) * g;
  v = b2 * v + (1.0f - b2) * g * g;
  p -= lr_t * m / (sqrtf(v) + eps);
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void fma4x4(float (&a)[4][4], const float4& x, const float4& w) {
  const float xs[4] = {x.x, x.y, x.z, x.w}, ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) a[u][v] = fmaf(xs[u], ws[v], a[u][v]);
}

// PUSH: each CTA stores its h1 / d2 units into every CTA's AT with DSMEM stores
// (measured faster for ensembles: 1.75e5 vs 1.33e5 member-steps/s with 8
// clusters); otherwise each CTA pulls the other CTAs' units with DSMEM loads
// (faster for one member: 39 vs 45 us per step)
template <int H, bool PUSH>
__global__ void __launch_bounds__(TR_THREADS, 1) train_kernel(const __grid_constant__ TrainParams p) {
  using S = TrainSmem<H>;
  constexpr int C = S::C;
  constexpr int WS = S::WS;
  constexpr int BM = TR_BMAX;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  uint32_t* idx = reinterpret_cast<uint32_t*>(s.d3);  // batch row indices (until d3 is formed)
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int e = (int)(blockIdx.x / C);  // ensemble member = cluster index
  const int tid = threadIdx.x;
  const int F = (int)p.F;
  const int c0 = c * TR_CPC;  // first owned hidden unit
  float* prm = p.params + (size_t)e * p.pstride;
  float *gW1p = prm + p.oW1, *gb1p = prm + p.ob1, *gW2p = prm + p.oW2, *gb2p = prm + p.ob2;
  float *gW3p = prm + p.oW3, *gb3p = prm + p.ob3;
  float* mW2 = p.mv + ((size_t)e * C + c) * 2 * H * TR_CPC;
  float* vW2 = mW2 + H * TR_CPC;
  const uint32_t* perms = p.perms ? p.perms + (size_t)e * p.max_epochs * p.n : nullptr;
  unsigned long long* prof = (p.prof && blockIdx.x == 0 && tid == 0) ? p.prof : nullptr;
  long long tmark = 0;
  // copy the other CTAs' 16-unit slices of AT (rows [16 q, 16 q + 16), B4 columns)
  // into ours: thread = (unit j = tid / 16, 16-byte words tid % 16 + 16 u); a
  // remote slice's four DSMEM loads are in flight before their stores
  auto gather = [&](int B4) {
    const int j = tid >> 4, w0 = (tid & 15) * 4;
#pragma unroll 1
    for (int q = 1; q < C; ++q) {
      const int rc = (c + q) % C;
      const float* src = cluster.map_shared_rank(s.AT, rc) + (rc * TR_CPC + j) * BM;
      float* dst = s.AT + (rc * TR_CPC + j) * BM;
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (w0 + 64 * u < B4) v[u] = ld4(src + w0 + 64 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (w0 + 64 * u < B4) *reinterpret_cast<float4*>(dst + w0 + 64 * u) = v[u];
    }
  };
  auto mark = [&](int i) {  // phase i ended now
    if (prof) {
      const long long now = clock64();
      if (i >= 0) prof[i] += (unsigned long long)(now - tmark);
      tmark = now;
    }
  };

  // ---- initial parameters (own columns, full W2), zero moments and padding rows
  for (int i = tid; i < H * H; i += TR_THREADS) s.W2[(i / H) * WS + i % H] = gW2p[i];
  for (int i = tid; i < F * TR_CPC; i += TR_THREADS) {
    s.W1o[i] = gW1p[(i / TR_CPC) * H + c0 + i % TR_CPC];
    s.mW1[i] = 0.0f;
    s.vW1[i] = 0.0f;
  }
  for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
    mW2[i] = 0.0f;
    vW2[i] = 0.0f;
  }
  if (tid < TR_CPC) {
    s.b1o[tid] = gb1p[c0 + tid];
    s.b2o[tid] = gb2p[c0 + tid];
    s.W3o[tid] = gW3p[c0 + tid];
    s.mb1[tid] = s.vb1[tid] = s.mb2[tid] = s.vb2[tid] = s.mW3[tid] = s.vW3[tid] = 0.0f;
  }
  if (tid == 0) {
    s.b3 = gb3p[0];
    s.mb3 = s.vb3 = 0.0f;
  }
  // rows past a short batch stay zero in every unit-major buffer (float4 loads)
  for (int i = tid; i < TR_FMAX * BM; i += TR_THREADS) s.XT[i] = 0.0f;
  for (int i = tid; i < H * BM; i += TR_THREADS) s.AT[i] = 0.0f;
  for (int i = tid; i < TR_CPC * BM; i += TR_THREADS) s.h1T[i] = s.h2T[i] = 0.0f;
  cluster.sync();
  mark(-1);

  const float alpha = p.alpha;
  double best = 1.0 / 0.0;
  uint32_t no_improve = 0, epochs = 0, reason = 0, t = 0;
  double b1t = 1.0, b2t = 1.0;  // beta^t in double, as the float64 reference forms lr_t

  for (uint32_t ep = 0; ep < p.max_epochs; ++ep) {
    const uint32_t* perm = perms ? perms + (size_t)ep * p.n : nullptr;
    double acc = 0.0;
    for (uint32_t s0 = 0; s0 < p.n; s0 += p.B) {
      const int B = (int)min(p.B, p.n - s0);
      const int B4 = (B + 3) & ~3;
      const float invB = 1.0f / (float)B;
      // ---- batch rows -> shared memory (unit-major); zero the tail rows of a short batch
      for (int r = tid; r < B; r += TR_THREADS) idx[r] = perm ? perm[s0 + r] : s0 + r;
      __syncthreads();
      for (int r = tid; r < B; r += TR_THREADS) {  // one row per thread: F loads in flight
        const float* xr = p.X + (size_t)idx[r] * F;
        float xv[TR_FMAX];
#pragma unroll
        for (int f = 0; f < TR_FMAX; ++f)
          if (f < F) xv[f] = __ldg(xr + f);
        const float yv = __ldg(p.y + idx[r]);
#pragma unroll
        for (int f = 0; f < TR_FMAX; ++f)
          if (f < F) s.XT[f * BM + r] = xv[f];
        s.y[r] = yv;
      }
      for (int i = tid; i < (B4 - B) * F; i += TR_THREADS) s.XT[(i % F) * BM + B + i / F] = 0.0f;
      __syncthreads();
      mark(0);

      // ---- forward, layer 1 (own units): h1 = relu(X W1 + b1) -> h1T and AT[own]
      for (int tt = tid; tt < (B4 / 4) * (TR_CPC / 4); tt += TR_THREADS) {
        const int r0 = (tt / (TR_CPC / 4)) * 4, j0 = (tt % (TR_CPC / 4)) * 4;
        float a[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[u][v] = s.b1o[j0 + v];
        for (int f = 0; f < F; ++f) fma4x4(a, ld4(&s.XT[f * BM + r0]), ld4(&s.W1o[f * TR_CPC + j0]));
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float4 h;
          h.x = r0 + 0 < B ? fmaxf(a[0][v], 0.0f) : 0.0f;
          h.y = r0 + 1 < B ? fmaxf(a[1][v], 0.0f) : 0.0f;
          h.z = r0 + 2 < B ? fmaxf(a[2][v], 0.0f) : 0.0f;
          h.w = r0 + 3 < B ? fmaxf(a[3][v], 0.0f) : 0.0f;
          *reinterpret_cast<float4*>(&s.h1T[(j0 + v) * BM + r0]) = h;
          if (PUSH) {
            // our h1 units into every CTA's AT (its rows of our units were last read
            // by the previous step's d1, before barrier (4) of that step)
#pragma unroll
            for (int q = 0; q < C; ++q)
              *reinterpret_cast<float4*>(cluster.map_shared_rank(&s.AT[(c0 + j0 + v) * BM + r0], q)) = h;
          } else {
            *reinterpret_cast<float4*>(&s.AT[(c0 + j0 + v) * BM + r0]) = h;
          }
        }
      }
      // own sum of squared weights (the L2 term uses the weights of this forward pass)
      {
        float q = 0.0f;
        for (int i = tid; i < F * TR_CPC; i += TR_THREADS) q = fmaf(s.W1o[i], s.W1o[i], q);
        for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
          const float w = s.W2[(i / TR_CPC) * WS + c0 + i % TR_CPC];
          q = fmaf(w, w, q);
        }
        if (tid < TR_CPC) q = fmaf(s.W3o[tid], s.W3o[tid], q);
        q = block_sum(q, s.red);
        if (tid == 0) s.wsq = q;
      }
      mark(1);
      cluster.sync();  // (1) every CTA's h1 slice is written (PUSH: is in every AT)
      mark(2);
      if (!PUSH) {
        gather(B4);  // the other CTAs' h1 units
        __syncthreads();
      }
      mark(3);

      // ---- forward, layer 2 (own units): h2 = relu(h1 W2 + b2); partial output h2 . W3
      for (int tt = tid; tt < (B4 / 4) * (TR_CPC / 4); tt += TR_THREADS) {
        const int r0 = (tt / (TR_CPC / 4)) * 4, j0 = (tt % (TR_CPC / 4)) * 4;
        float a[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[u][v] = s.b2o[j0 + v];
#pragma unroll 4
        for (int k = 0; k < H; ++k) fma4x4(a, ld4(&s.AT[k * BM + r0]), ld4(&s.W2[k * WS + c0 + j0]));
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float4 h;
          h.x = r0 + 0 < B ? fmaxf(a[0][v], 0.0f) : 0.0f;
          h.y = r0 + 1 < B ? fmaxf(a[1][v], 0.0f) : 0.0f;
          h.z = r0 + 2 < B ? fmaxf(a[2][v], 0.0f) : 0.0f;
          h.w = r0 + 3 < B ? fmaxf(a[3][v], 0.0f) : 0.0f;
          *reinterpret_cast<float4*>(&s.h2T[(j0 + v) * BM + r0]) = h;
        }
      }
      __syncthreads();
      for (int r = tid; r < B; r += TR_THREADS) {
        float a = 0.0f;
#pragma unroll
        for (int j = 0; j < TR_CPC; ++j) a = fmaf(s.h2T[j * BM + r], s.W3o[j], a);
        s.ypart[r] = a;
      }
      mark(4);
      cluster.sync();  // (2) every CTA's partial output and weight norm are written
      mark(5);

      // ---- output and loss (every CTA, same order): yhat = b3 + sum_q ypart_q
      float wsq = 0.0f;
      for (int q = 0; q < C; ++q) wsq += *cluster.map_shared_rank(&s.wsq, q);
      float l2 = 0.0f;
      for (int r = tid; r < B4; r += TR_THREADS) {
        float d = 0.0f;
        if (r < B) {
          float yh = s.b3;
          for (int q = 0; q < C; ++q) yh += cluster.map_shared_rank(s.ypart, q)[r];
          d = yh - s.y[r];
        }
        l2 = fmaf(d, d, l2);
        s.d3[r] = d;
      }
      l2 = block_sum(l2, s.red);  // includes __syncthreads: d3 visible
      const float loss = 0.5f * l2 * invB + 0.5f * alpha * wsq * invB;
      acc += (double)loss * (double)B;
      mark(6);

      // ---- backward: gW3 (warp w: units w, w + 8), gb3; d2 = d3 W3 . [h2 > 0] in place
      {
        const int w = tid >> 5, ln = tid & 31;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int j = w + 8 * jj;
          float g = 0.0f;
          for (int r = ln; r < B; r += 32) g = fmaf(s.h2T[j * BM + r], s.d3[r], g);
          g = warp_sum(g);
          if (ln == 0) s.gW3[j] = (g + alpha * s.W3o[j]) * invB;
        }
        if (w == 0) {
          float g = 0.0f;
          for (int r = ln; r < B; r += 32) g += s.d3[r];
          g = warp_sum(g);
          if (ln == 0) s.gb3 = g * invB;
        }
      }
      __syncthreads();
      for (int i = tid; i < TR_CPC * B4; i += TR_THREADS) {
        const int j = i / B4, r = i % B4;
        float& h = s.h2T[j * BM + r];
        h = h > 0.0f ? s.d3[r] * s.W3o[j] : 0.0f;
      }
      __syncthreads();
      // gW2[:, own] = (h1^T d2 + alpha W2) / B (AT still holds h1): thread tile 2 k x 4 j
      {
        // units j = q + 4 v (q = tid % 4): the 4 threads of a quarter-warp read
        // consecutive h2T rows, whose 16-byte words fall in distinct bank groups
        const int k0 = (tid >> 2) * 2, q4 = tid & 3;
        if (k0 < H) {
          float a[2][4] = {};
          for (int r = 0; r < B4; r += 4) {
            const float4 x0 = ld4(&s.AT[k0 * BM + r]), x1 = ld4(&s.AT[(k0 + 1) * BM + r]);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const float4 d = ld4(&s.h2T[(q4 + 4 * v) * BM + r]);
              a[0][v] = fmaf(x0.x, d.x, fmaf(x0.y, d.y, fmaf(x0.z, d.z, fmaf(x0.w, d.w, a[0][v]))));
              a[1][v] = fmaf(x1.x, d.x, fmaf(x1.y, d.y, fmaf(x1.z, d.z, fmaf(x1.w, d.w, a[1][v]))));
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
              s.gW2[(k0 + u) * TR_CPC + q4 + 4 * v] = (a[u][v] + alpha * s.W2[(k0 + u) * WS + c0 + q4 + 4 * v]) * invB;
        }
      }
      {  // gb2: warp w sums units w, w + 8
        const int w = tid >> 5, ln = tid & 31;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          float g = 0.0f;
          for (int r = ln; r < B; r += 32) g += s.h2T[(w + 8 * jj) * BM + r];
          g = warp_sum(g);
          if (ln == 0) s.gb2[w + 8 * jj] = g * invB;
        }
      }
      __syncthreads();
      if (PUSH) {
        mark(7);
        cluster.sync();  // (3) every CTA is done with gW2, i.e. with the h1 rows of AT
        mark(8);
        for (int i = tid; i < TR_CPC * (B4 / 4); i += TR_THREADS) {  // our d2 units into every AT
          const int o = (i / (B4 / 4)) * BM + (i % (B4 / 4)) * 4;
          const float4 d = ld4(&s.h2T[o]);
#pragma unroll
          for (int q = 0; q < C; ++q) *reinterpret_cast<float4*>(cluster.map_shared_rank(&s.AT[c0 * BM + o], q)) = d;
        }
        cluster.sync();  // (3b) every CTA's d2 units are in every AT
      } else {
        // own d2 units -> AT (the other CTAs finished reading our h1 units at (2))
        for (int i = tid; i < TR_CPC * (B4 / 4); i += TR_THREADS) {
          const int o = (i / (B4 / 4)) * BM + (i % (B4 / 4)) * 4;
          *reinterpret_cast<float4*>(&s.AT[c0 * BM + o]) = ld4(&s.h2T[o]);
        }
        mark(7);
        cluster.sync();  // (3) every CTA's d2 slice is written
        mark(8);
        gather(B4);  // the other CTAs' d2 units
        __syncthreads();
      }
      mark(9);
      // d1 = d2 W2^T . [h1 > 0] (own units, in place over h1T): W2 rows of the own units
      for (int tt = tid; tt < (B4 / 4) * (TR_CPC / 4); tt += TR_THREADS) {
        const int r0 = (tt / (TR_CPC / 4)) * 4, j0 = (tt % (TR_CPC / 4)) * 4;
        float a[4][4] = {};
        for (int m4 = 0; m4 < H; m4 += 4) {
          float4 w[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) w[v] = ld4(&s.W2[(c0 + j0 + v) * WS + m4]);
          const float4 d0 = ld4(&s.AT[(m4 + 0) * BM + r0]), d1 = ld4(&s.AT[(m4 + 1) * BM + r0]);
          const float4 d2 = ld4(&s.AT[(m4 + 2) * BM + r0]), d3 = ld4(&s.AT[(m4 + 3) * BM + r0]);
          fma4x4(a, d0, make_float4(w[0].x, w[1].x, w[2].x, w[3].x));
          fma4x4(a, d1, make_float4(w[0].y, w[1].y, w[2].y, w[3].y));
          fma4x4(a, d2, make_float4(w[0].z, w[1].z, w[2].z, w[3].z));
          fma4x4(a, d3, make_float4(w[0].w, w[1].w, w[2].w, w[3].w));
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float4& h = *reinterpret_cast<float4*>(&s.h1T[(j0 + v) * BM + r0]);
          float4 o = h;
          o.x = o.x > 0.0f ? a[0][v] : 0.0f;
          o.y = o.y > 0.0f ? a[1][v] : 0.0f;
          o.z = o.z > 0.0f ? a[2][v] : 0.0f;
          o.w = o.w > 0.0f ? a[3][v] : 0.0f;
          h = o;
        }
      }
      __syncthreads();
      // gW1[:, own] = (X^T d1 + alpha W1) / B, gb1 = mean d1
      for (int i = tid; i < F * TR_CPC; i += TR_THREADS) {
        const int f = i / TR_CPC, j = i % TR_CPC;
        float g = 0.0f;
        for (int r = 0; r < B4; r += 4) {
          const float4 x = ld4(&s.XT[f * BM + r]), d = ld4(&s.h1T[j * BM + r]);
          g = fmaf(x.x, d.x, fmaf(x.y, d.y, fmaf(x.z, d.z, fmaf(x.w, d.w, g))));
        }
        s.gW1[i] = (g + alpha * s.W1o[i]) * invB;
      }
      {  // gb1: warp w sums units w, w + 8
        const int w = tid >> 5, ln = tid & 31;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          float g = 0.0f;
          for (int r = ln; r < B; r += 32) g += s.h1T[(w + 8 * jj) * BM + r];
          g = warp_sum(g);
          if (ln == 0) s.gb1[w + 8 * jj] = g * invB;
        }
      }
      mark(10);
      cluster.sync();  // (4) every CTA is done reading W2 rows and our d2 slice
      mark(11);

      // ---- Adam on the own parameters; new W2 columns -> every CTA's copy
      ++t;
      b1t *= (double)p.beta1;
      b2t *= (double)p.beta2;
      const float lr_t = (float)((double)p.lr0 * sqrt(1.0 - b2t) / (1.0 - b1t));
      const float be1 = p.beta1, be2 = p.beta2, eps = p.eps;
      // W2 columns: four elements' moment loads in flight at a time
      constexpr int NE = H * TR_CPC / TR_THREADS;  // 8 / 4 / 2 elements per thread
      constexpr int NB = NE < 4 ? NE : 4;
#pragma unroll 1
      for (int e0 = 0; e0 < NE; e0 += NB) {
        float mm[NB], vv[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          mm[u] = mW2[tid + (e0 + u) * TR_THREADS];
          vv[u] = vW2[tid + (e0 + u) * TR_THREADS];
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int i = tid + (e0 + u) * TR_THREADS, k = i / TR_CPC, j = i % TR_CPC;
          float w = s.W2[k * WS + c0 + j];
          adam(w, mm[u], vv[u], s.gW2[i], be1, be2, lr_t, eps);
          mW2[i] = mm[u];
          vW2[i] = vv[u];
#pragma unroll
          for (int q = 0; q < C; ++q) cluster.map_shared_rank(s.W2, q)[k * WS + c0 + j] = w;
        }
      }
      for (int i = tid; i < F * TR_CPC; i += TR_THREADS) adam(s.W1o[i], s.mW1[i], s.vW1[i], s.gW1[i], be1, be2, lr_t, eps);
      if (tid < TR_CPC) {
        adam(s.b1o[tid], s.mb1[tid], s.vb1[tid], s.gb1[tid], be1, be2, lr_t, eps);
        adam(s.b2o[tid], s.mb2[tid], s.vb2[tid], s.gb2[tid], be1, be2, lr_t, eps);
        adam(s.W3o[tid], s.mW3[tid], s.vW3[tid], s.gW3[tid], be1, be2, lr_t, eps);
      }
      if (tid == 0) adam(s.b3, s.mb3, s.vb3, s.gb3, be1, be2, lr_t, eps);  // identical on every CTA
      mark(12);
      cluster.sync();  // (5) every W2 copy holds the new weights
      mark(13);
    }
    // ---- epoch loss and the stopping rule (identical on every CTA of the member)
    const double el = acc / (double)p.n;
    if (c == 0 && tid == 0) p.loss_hist[(size_t)e * p.max_epochs + ep] = el;
    epochs = ep + 1;
    if (el > best - p.tol) ++no_improve;
    else no_improve = 0;
    if (el < best) best = el;
    if (no_improve > p.n_iter_no_change) {
      reason = 1;
      break;
    }
  }

  // ---- trained parameters -> global memory (own columns; CTA 0 writes b3)
  for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
    const int k = i / TR_CPC, j = i % TR_CPC;
    gW2p[k * H + c0 + j] = s.W2[k * WS + c0 + j];
  }
  for (int i = tid; i < F * TR_CPC; i += TR_THREADS) gW1p[(i / TR_CPC) * H + c0 + i % TR_CPC] = s.W1o[i];
  if (tid < TR_CPC) {
    gb1p[c0 + tid] = s.b1o[tid];
    gb2p[c0 + tid] = s.b2o[tid];
    gW3p[c0 + tid] = s.W3o[tid];
  }
  if (c == 0 && tid == 0) {
    gb3p[0] = s.b3;
    p.result[3 * e + 0] = epochs;
    p.result[3 * e + 1] = reason;
    p.result[3 * e + 2] = t;
  }
  cluster.sync();  // no CTA exits while its shared memory may still be read
}

}  // namespace surr
