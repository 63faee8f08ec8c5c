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
// B200 mapping: the whole run is ONE launch of a thread-block cluster of
// C = H / 16 CTAs (8 at H = 128) that stays resident for every epoch.  CTA c
// owns the 16 hidden units [16c, 16c + 16) of both hidden layers: its columns
// of W1, W2, W3 and their Adam state, and computes those units' activations and
// deltas for the whole batch.  Layers meet through distributed shared memory:
// each CTA gathers the other CTAs' 16-column slices of h1 (forward) and of d2
// (backward) into its own full-width buffer, the output is a cluster reduction
// of per-CTA partial dot products, and the updated W2 columns are written into
// every CTA's full W2 copy (needed by d1 = d2 W2^T).  Five cluster barriers
// per step; no global-memory traffic except the batch rows and the W2 Adam
// moments.  FP32 FMA throughout (the step is ~10 MFLOP: latency-bound, not a
// tensor-core contraction worth splitting into 3xFP16).
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

namespace surr {

namespace cg = cooperative_groups;

constexpr int TR_BMAX = 200;  // batch rows held in shared memory (the paper's batch size)
constexpr int TR_FMAX = 24;   // input features (14 parameters + device features)
constexpr int TR_CPC = 16;    // hidden units per CTA
constexpr int TR_THREADS = 256;

struct TrainParams {
  const float* X;         // [n][F] standardised inputs
  const float* y;         // [n] standardised targets
  const uint32_t* perms;  // [max_epochs][n] epoch permutations (null: identity order)
  uint32_t n, F, B;       // rows, features, batch size
  uint32_t max_epochs, n_iter_no_change;
  float alpha, beta1, beta2, lr0, eps;
  double tol;
  // parameters, fp32, row-major fan_in x fan_out: in = initial, out = trained
  float *W1, *b1, *W2, *b2, *W3, *b3;  // [F][H], [H], [H][H], [H], [H], [1]
  float* mv;                           // Adam moments of this CTA's W2 columns: [C][2][H][16]
  double* loss_hist;                   // [max_epochs]
  uint32_t* result;                    // [0] epochs run, [1] stop reason (0 max_epochs, 1 tol), [2] Adam steps
};

template <int H>
struct TrainSmem {
  static constexpr int C = H / TR_CPC;
  float W2[H * H];              // full copy, row-major [k][n]
  float A[TR_BMAX * H];         // h1 (forward), then d2 (backward), all H columns
  float h1o[TR_BMAX * TR_CPC];  // own h1 columns, then d1 in place
  float h2o[TR_BMAX * TR_CPC];  // own h2 columns, then d2 in place
  float X[TR_BMAX * TR_FMAX];
  float y[TR_BMAX];
  float ypart[TR_BMAX];         // own partial of yhat (read by every CTA)
  float gW2[H * TR_CPC];        // gradient of own W2 columns
  float W1o[TR_FMAX * TR_CPC], gW1[TR_FMAX * TR_CPC], mW1[TR_FMAX * TR_CPC], vW1[TR_FMAX * TR_CPC];
  float b1o[TR_CPC], b2o[TR_CPC], W3o[TR_CPC], gb1[TR_CPC], gb2[TR_CPC], gW3[TR_CPC];
  float mb1[TR_CPC], vb1[TR_CPC], mb2[TR_CPC], vb2[TR_CPC], mW3[TR_CPC], vW3[TR_CPC];
  float wsq;                    // own sum of squared weights (read by every CTA)
  float red[TR_THREADS / 32];
  float b3, mb3, vb3;
  uint32_t idx[TR_BMAX];        // batch row indices
};

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
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

template <int H>
__global__ void __launch_bounds__(TR_THREADS, 1) train_kernel(const __grid_constant__ TrainParams p) {
  using S = TrainSmem<H>;
  constexpr int C = S::C;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int F = (int)p.F;
  const int c0 = c * TR_CPC;  // first owned hidden unit
  float* mW2 = p.mv + (size_t)c * 2 * H * TR_CPC;
  float* vW2 = mW2 + H * TR_CPC;

  // ---- load the initial parameters (own columns, full W2) and zero the moments
  for (int i = tid; i < H * H; i += TR_THREADS) s.W2[i] = p.W2[i];
  for (int i = tid; i < F * TR_CPC; i += TR_THREADS) {
    s.W1o[i] = p.W1[(i / TR_CPC) * H + c0 + i % TR_CPC];
    s.mW1[i] = 0.0f;
    s.vW1[i] = 0.0f;
  }
  for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
    mW2[i] = 0.0f;
    vW2[i] = 0.0f;
  }
  if (tid < TR_CPC) {
    s.b1o[tid] = p.b1[c0 + tid];
    s.b2o[tid] = p.b2[c0 + tid];
    s.W3o[tid] = p.W3[c0 + tid];
    s.mb1[tid] = s.vb1[tid] = s.mb2[tid] = s.vb2[tid] = s.mW3[tid] = s.vW3[tid] = 0.0f;
  }
  if (tid == 0) {
    s.b3 = p.b3[0];
    s.mb3 = s.vb3 = 0.0f;
  }
  cluster.sync();

  const float alpha = p.alpha;
  double best = 1.0 / 0.0;
  uint32_t no_improve = 0, epochs = 0, reason = 0, t = 0;
  double b1t = 1.0, b2t = 1.0;  // beta^t in double, as the float64 reference forms lr_t

  for (uint32_t ep = 0; ep < p.max_epochs; ++ep) {
    const uint32_t* perm = p.perms ? p.perms + (size_t)ep * p.n : nullptr;
    double acc = 0.0;
    for (uint32_t s0 = 0; s0 < p.n; s0 += p.B) {
      const int B = (int)min(p.B, p.n - s0);
      const float invB = 1.0f / (float)B;
      // ---- batch rows -> shared memory
      for (int r = tid; r < B; r += TR_THREADS) s.idx[r] = perm ? perm[s0 + r] : s0 + r;
      __syncthreads();
      for (int i = tid; i < B * F; i += TR_THREADS) {
        const int r = i / F, f = i % F;
        s.X[r * TR_FMAX + f] = p.X[(size_t)s.idx[r] * F + f];
      }
      for (int r = tid; r < B; r += TR_THREADS) s.y[r] = p.y[s.idx[r]];
      __syncthreads();

      // ---- forward, layer 1 (own units): h1 = relu(X W1 + b1) -> A[:, own] and h1o
      for (int i = tid; i < B * TR_CPC; i += TR_THREADS) {
        const int r = i / TR_CPC, j = i % TR_CPC;
        float a = s.b1o[j];
        for (int f = 0; f < F; ++f) a = fmaf(s.X[r * TR_FMAX + f], s.W1o[f * TR_CPC + j], a);
        a = fmaxf(a, 0.0f);
        s.h1o[i] = a;
        s.A[r * H + c0 + j] = a;
      }
      // own sum of squared weights (the L2 term uses the weights of this forward pass)
      {
        float q = 0.0f;
        for (int i = tid; i < F * TR_CPC; i += TR_THREADS) q = fmaf(s.W1o[i], s.W1o[i], q);
        for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
          const float w = s.W2[(i / TR_CPC) * H + c0 + i % TR_CPC];
          q = fmaf(w, w, q);
        }
        if (tid < TR_CPC) q = fmaf(s.W3o[tid], s.W3o[tid], q);
        q = block_sum(q, s.red);
        if (tid == 0) s.wsq = q;
      }
      cluster.sync();  // (1) every CTA's h1 slice is written
      // gather the other CTAs' h1 slices (16-byte DSMEM loads)
      for (int q = 1; q < C; ++q) {
        const int rc = (c + q) % C;
        const float* rA = cluster.map_shared_rank(s.A, rc);
        for (int i = tid; i < B * (TR_CPC / 4); i += TR_THREADS) {
          const int r = i / (TR_CPC / 4), v4 = i % (TR_CPC / 4);
          const int o = r * H + rc * TR_CPC + v4 * 4;
          *reinterpret_cast<float4*>(&s.A[o]) = *reinterpret_cast<const float4*>(&rA[o]);
        }
      }
      __syncthreads();

      // ---- forward, layer 2 (own units): h2 = relu(h1 W2 + b2); partial output h2 . W3
      // thread tile: 4 rows x 4 units (B x 16 outputs -> up to 200 tiles)
      for (int tt = tid; tt < ((B + 3) / 4) * (TR_CPC / 4); tt += TR_THREADS) {
        const int r0 = (tt / (TR_CPC / 4)) * 4, j0 = (tt % (TR_CPC / 4)) * 4;
        float a[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[u][v] = s.b2o[j0 + v];
        for (int k = 0; k < H; ++k) {
          const float4 w = *reinterpret_cast<const float4*>(&s.W2[k * H + c0 + j0]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float x = (r0 + u < B) ? s.A[(r0 + u) * H + k] : 0.0f;
            a[u][0] = fmaf(x, w.x, a[u][0]);
            a[u][1] = fmaf(x, w.y, a[u][1]);
            a[u][2] = fmaf(x, w.z, a[u][2]);
            a[u][3] = fmaf(x, w.w, a[u][3]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r0 + u < B)
#pragma unroll
            for (int v = 0; v < 4; ++v) s.h2o[(r0 + u) * TR_CPC + j0 + v] = fmaxf(a[u][v], 0.0f);
      }
      __syncthreads();
      for (int r = tid; r < B; r += TR_THREADS) {
        float a = 0.0f;
#pragma unroll
        for (int j = 0; j < TR_CPC; ++j) a = fmaf(s.h2o[r * TR_CPC + j], s.W3o[j], a);
        s.ypart[r] = a;
      }
      cluster.sync();  // (2) every CTA's partial output and weight norm are written

      // ---- output and loss (every CTA, same order): yhat = b3 + sum_q ypart_q
      float wsq = 0.0f;
      for (int q = 0; q < C; ++q) wsq += *cluster.map_shared_rank(&s.wsq, q);
      float l2 = 0.0f;
      for (int r = tid; r < B; r += TR_THREADS) {
        float yh = s.b3;
        for (int q = 0; q < C; ++q) yh += cluster.map_shared_rank(s.ypart, q)[r];
        const float d = yh - s.y[r];
        l2 = fmaf(d, d, l2);
        s.idx[r] = __float_as_uint(d);  // d3 (the row indices are no longer needed)
      }
      l2 = block_sum(l2, s.red);  // includes __syncthreads: d3 visible
      const float loss = 0.5f * l2 * invB + 0.5f * alpha * wsq * invB;
      acc += (double)loss * (double)B;
      const float* d3 = reinterpret_cast<const float*>(s.idx);

      // ---- backward: gW3, gb3; d2 = d3 W3 . [h2 > 0] in place (own units)
      if (tid < TR_CPC) {
        float g = 0.0f;
        for (int r = 0; r < B; ++r) g = fmaf(s.h2o[r * TR_CPC + tid], d3[r], g);
        s.gW3[tid] = (g + alpha * s.W3o[tid]) * invB;
      }
      float gb3 = 0.0f;
      {
        float g = 0.0f;
        for (int r = tid; r < B; r += TR_THREADS) g += d3[r];
        gb3 = block_sum(g, s.red) * invB;  // barrier: gW3 read h2o before it is overwritten
      }
      for (int i = tid; i < B * TR_CPC; i += TR_THREADS) {
        const int r = i / TR_CPC, j = i % TR_CPC;
        s.h2o[i] = s.h2o[i] > 0.0f ? d3[r] * s.W3o[j] : 0.0f;
      }
      __syncthreads();
      // gW2[:, own] = (h1^T d2 + alpha W2) / B (A still holds h1), gb2 = mean d2
      for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
        const int k = i / TR_CPC, j = i % TR_CPC;
        float g = 0.0f;
        for (int r = 0; r < B; ++r) g = fmaf(s.A[r * H + k], s.h2o[r * TR_CPC + j], g);
        s.gW2[i] = (g + alpha * s.W2[k * H + c0 + j]) * invB;
      }
      if (tid < TR_CPC) {
        float g = 0.0f;
        for (int r = 0; r < B; ++r) g += s.h2o[r * TR_CPC + tid];
        s.gb2[tid] = g * invB;
      }
      __syncthreads();
      // own d2 slice -> A (the other CTAs finished reading our h1 slice at (2))
      for (int i = tid; i < B * TR_CPC; i += TR_THREADS) s.A[(i / TR_CPC) * H + c0 + i % TR_CPC] = s.h2o[i];
      cluster.sync();  // (3) every CTA's d2 slice is written
      for (int q = 1; q < C; ++q) {
        const int rc = (c + q) % C;
        const float* rA = cluster.map_shared_rank(s.A, rc);
        for (int i = tid; i < B * (TR_CPC / 4); i += TR_THREADS) {
          const int r = i / (TR_CPC / 4), v4 = i % (TR_CPC / 4);
          const int o = r * H + rc * TR_CPC + v4 * 4;
          *reinterpret_cast<float4*>(&s.A[o]) = *reinterpret_cast<const float4*>(&rA[o]);
        }
      }
      __syncthreads();
      // d1 = d2 W2^T . [h1 > 0] (own units, in place over h1o): W2 rows of the own units
      for (int tt = tid; tt < ((B + 3) / 4) * (TR_CPC / 4); tt += TR_THREADS) {
        const int r0 = (tt / (TR_CPC / 4)) * 4, j0 = (tt % (TR_CPC / 4)) * 4;
        float a[4][4] = {};
        for (int m4 = 0; m4 < H; m4 += 4) {
          float4 w[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) w[v] = *reinterpret_cast<const float4*>(&s.W2[(c0 + j0 + v) * H + m4]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (r0 + u >= B) break;
            const float4 d = *reinterpret_cast<const float4*>(&s.A[(r0 + u) * H + m4]);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              a[u][v] = fmaf(d.x, w[v].x, a[u][v]);
              a[u][v] = fmaf(d.y, w[v].y, a[u][v]);
              a[u][v] = fmaf(d.z, w[v].z, a[u][v]);
              a[u][v] = fmaf(d.w, w[v].w, a[u][v]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r0 + u < B)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float& h = s.h1o[(r0 + u) * TR_CPC + j0 + v];
              h = h > 0.0f ? a[u][v] : 0.0f;
            }
      }
      __syncthreads();
      // gW1[:, own] = (X^T d1 + alpha W1) / B, gb1 = mean d1
      for (int i = tid; i < F * TR_CPC; i += TR_THREADS) {
        const int f = i / TR_CPC, j = i % TR_CPC;
        float g = 0.0f;
        for (int r = 0; r < B; ++r) g = fmaf(s.X[r * TR_FMAX + f], s.h1o[r * TR_CPC + j], g);
        s.gW1[i] = (g + alpha * s.W1o[i]) * invB;
      }
      if (tid < TR_CPC) {
        float g = 0.0f;
        for (int r = 0; r < B; ++r) g += s.h1o[r * TR_CPC + tid];
        s.gb1[tid] = g * invB;
      }
      cluster.sync();  // (4) every CTA is done reading W2 rows and our d2 slice

      // ---- Adam on the own parameters; new W2 columns -> every CTA's copy
      ++t;
      b1t *= (double)p.beta1;
      b2t *= (double)p.beta2;
      const float lr_t = (float)((double)p.lr0 * sqrt(1.0 - b2t) / (1.0 - b1t));
      const float be1 = p.beta1, be2 = p.beta2, eps = p.eps;
      for (int i = tid; i < H * TR_CPC; i += TR_THREADS) {
        const int k = i / TR_CPC, j = i % TR_CPC;
        float w = s.W2[k * H + c0 + j], m = mW2[i], v = vW2[i];
        adam(w, m, v, s.gW2[i], be1, be2, lr_t, eps);
        mW2[i] = m;
        vW2[i] = v;
        for (int q = 0; q < C; ++q) cluster.map_shared_rank(s.W2, q)[k * H + c0 + j] = w;
      }
      for (int i = tid; i < F * TR_CPC; i += TR_THREADS) adam(s.W1o[i], s.mW1[i], s.vW1[i], s.gW1[i], be1, be2, lr_t, eps);
      if (tid < TR_CPC) {
        adam(s.b1o[tid], s.mb1[tid], s.vb1[tid], s.gb1[tid], be1, be2, lr_t, eps);
        adam(s.b2o[tid], s.mb2[tid], s.vb2[tid], s.gb2[tid], be1, be2, lr_t, eps);
        adam(s.W3o[tid], s.mW3[tid], s.vW3[tid], s.gW3[tid], be1, be2, lr_t, eps);
      }
      if (tid == 0) adam(s.b3, s.mb3, s.vb3, gb3, be1, be2, lr_t, eps);  // identical on every CTA
      cluster.sync();  // (5) every W2 copy holds the new weights
    }
    // ---- epoch loss and the stopping rule (identical on every CTA)
    const double el = acc / (double)p.n;
    if (c == 0 && tid == 0) p.loss_hist[ep] = el;
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
    p.W2[k * H + c0 + j] = s.W2[k * H + c0 + j];
  }
  for (int i = tid; i < F * TR_CPC; i += TR_THREADS) p.W1[(i / TR_CPC) * H + c0 + i % TR_CPC] = s.W1o[i];
  if (tid < TR_CPC) {
    p.b1[c0 + tid] = s.b1o[tid];
    p.b2[c0 + tid] = s.b2o[tid];
    p.W3[c0 + tid] = s.W3o[tid];
  }
  if (c == 0 && tid == 0) {
    p.b3[0] = s.b3;
    p.result[0] = epochs;
    p.result[1] = reason;
    p.result[2] = t;
  }
  cluster.sync();  // no CTA exits while its shared memory may still be read
}

}  // namespace surr
