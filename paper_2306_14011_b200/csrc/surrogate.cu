// Host runtime and C ABI of the B200 surrogate sweep (include/surrogate.h).
//
// Responsibilities: validate descriptors, compute |S| and
// the decoder's super-digit radices and per-tile stride digits, build the value lookup table
// (StandardScaler applied in double, then rounded to the
// operand format), fold b_1 / device features / y de-standardisation into the
// layer parameters, pack the UMMA shared-memory image, own device buffers and
// launch K1 (sweep_kernel), K2 (merge_kernel) and K3 (sweep_kernel in predict
// mode).  No arithmetic of the method runs here per config: every config is
// evaluated by the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sweep_kernel.cuh"
#include "sweep_kernel3.cuh"
#include "sweep_kernel5.cuh"
#include "sweep_kernel6.cuh"
#include "sweep_kernel8.cuh"
#include "sweep_kernel8e.cuh"
#include "sweep_kernel_pair.cuh"
#include "train_kernel.cuh"
#ifndef SURR_PAIR_NSUB
#define SURR_PAIR_NSUB 2
#endif

using namespace surr;

// Device copies of a host image that kernels read by pointer (the value table,
// the weight image): two slots used alternately.  A slot is rewritten only
// after the events recorded behind every launch that read it (one per launch
// stream) and behind its own upload have completed, so replacing a table never
// synchronises the device and never changes bytes a queued sweep still reads.
struct UploadRing {
  void* d[2] = {nullptr, nullptr};
  void* hpin[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> users[2];
  int cur = -1;
};

struct surrogate {
  int dev = -1;
  int sms = 0;
  std::string err;
  // model
  bool loaded = false;
  int prec = 0;
  uint32_t H = 0, NL = 0, P = 0;
  std::vector<uint8_t> wimg;
  UploadRing wring;  // device weight image (all members), two slots
  KParams mp{};  // model part of the kernel parameters (member 0)
  std::vector<KParams> members;  // per-member model parameters (ensemble)
  float* d_acc = nullptr;        // ensemble accumulation buffer (fp32 per config of a chunk)
  size_t d_acc_cap = 0;
  std::vector<double> hshift, hscale;  // host copies of the input affine map
  // FP16-operand precisions: per member, the layer-1 operand [W1; b1'] (K0 x H)
  // and the hidden->hidden layers whose outputs feed another UMMA, for the
  // range bound checked against each space (f16_range_check)
  std::vector<std::vector<double>> rb_B1;
  std::vector<std::vector<std::vector<double>>> rb_W, rb_b;
  // space cache
  bool space_valid = false;
  std::vector<uint32_t> c_radix;
  std::vector<double> c_values;
  std::vector<uint8_t> lut;
  UploadRing lring;  // device value table, two slots
  KParams sp{};  // space part (decoder) of the kernel parameters
  uint64_t card = 0;
  uint32_t spg = 2;  // parameter slots per decoder group of the cached table
  // buffers
  surr_record* d_recs = nullptr;
  size_t d_recs_cap = 0;
  surr_record* d_merged = nullptr;
  uint64_t* d_idx = nullptr;
  float* d_t = nullptr;
  uint32_t* d_ctr = nullptr;    // tickets of the fused grid merge tree (zero between launches)
  uint32_t* a0_dump = nullptr;  // MODE_A0 output of the current call
  uint64_t a0_stride = 1;
  // debug timeline
  unsigned long long* trace = nullptr;
  uint32_t trace_n = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  uint32_t launches = 0;
};

namespace {

thread_local std::string g_err;

surr_status fail(surrogate* h, surr_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf; else g_err = buf;
  return st;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return fail(h, SURR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// record "slot cur of the ring was read by work queued on st up to here"
surr_status ring_mark_use(surrogate* h, UploadRing& r, cudaStream_t st) {
  if (r.cur < 0) return SURR_OK;
  auto& u = r.users[r.cur];
  cudaEvent_t ev = nullptr;
  for (auto& e : u)
    if (e.first == st) ev = e.second;
  if (!ev) {
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    u.emplace_back(st, ev);
  }
  CU(cudaEventRecord(ev, st));
  return SURR_OK;
}

// upload `bytes` of host data into the ring's other slot; stream-ordered on st
// (async from pinned memory) or, with sync, complete on return.  *out = device copy.
surr_status ring_upload(surrogate* h, UploadRing& r, const void* data, size_t bytes, cudaStream_t st, bool sync,
                        void** out) {
  const int s = (r.cur + 1) & 1;
  for (auto& e : r.users[s]) CU(cudaEventSynchronize(e.second));  // its last readers and upload are done
  if (bytes > r.cap[s]) {
    if (r.d[s]) cudaFree(r.d[s]);
    if (r.hpin[s]) cudaFreeHost(r.hpin[s]);
    r.d[s] = r.hpin[s] = nullptr;
    r.cap[s] = 0;
    if (cudaMalloc(&r.d[s], bytes) != cudaSuccess || cudaMallocHost(&r.hpin[s], bytes) != cudaSuccess)
      return fail(h, SURR_E_OOM, "cudaMalloc upload slot (%zu B)", bytes);
    r.cap[s] = bytes;
  }
  memcpy(r.hpin[s], data, bytes);
  if (sync) {
    CU(cudaMemcpy(r.d[s], r.hpin[s], bytes, cudaMemcpyHostToDevice));
  } else {
    CU(cudaMemcpyAsync(r.d[s], r.hpin[s], bytes, cudaMemcpyHostToDevice, st));
  }
  r.cur = s;
  surr_status rc = ring_mark_use(h, r, st);  // the pinned staging copy is in use until the copy ran
  if (rc) return rc;
  *out = r.d[s];
  return SURR_OK;
}

void ring_free(UploadRing& r) {
  for (int s = 0; s < 2; ++s) {
    for (auto& e : r.users[s]) { cudaEventSynchronize(e.second); cudaEventDestroy(e.second); }
    r.users[s].clear();
    if (r.d[s]) cudaFree(r.d[s]);
    if (r.hpin[s]) cudaFreeHost(r.hpin[s]);
    r.d[s] = r.hpin[s] = nullptr;
  }
}

// ------------------------------------------------------------ rounding (host)
uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
uint16_t bf16_rne(float f) {  // same as __float2bfloat16_rn for finite values
  uint32_t u = f32_bits(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
// IEEE binary16, round to nearest even, with subnormals (same as cvt.rn.f16.f32)
uint16_t f16_rne(float f) {
  const uint32_t u = f32_bits(f);
  const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
  const uint32_t a = u & 0x7FFFFFFFu;
  if (a > 0x7F800000u) return sign | 0x7E00u;
  if (a >= 0x477FF000u) return sign | 0x7C00u;  // >= 65520 rounds to inf
  if (a >= 0x38800000u) {                          // normal half (>= 2^-14)
    const uint32_t r = (a + 0xFFFu + ((a >> 13) & 1u)) >> 13;
    return sign | (uint16_t)(r - (112u << 10));
  }
  return sign | (uint16_t)std::nearbyint((double)bits_f32(a) * 16777216.0);  // multiples of 2^-24
}
// the 16-bit operand format of a kind::f16 precision
uint16_t h16_rne(int prec, float f) { return prec == PREC_BF16 ? bf16_rne(f) : f16_rne(f); }
uint32_t tf32_rn(float f) {  // same as cvt.rn.tf32.f32 (nearest even) for finite values
  uint32_t u = f32_bits(f);
  if ((u & 0x7FFFFFFFu) >= 0x7F800000u) return u;
  return (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
}
// hi = tf32(x), lo = fp32(x) - hi exactly (the UMMA reads lo's top 19 bits)
void tf32_split(double x, uint32_t* hi, uint32_t* lo) {
  float f = (float)x;
  *hi = tf32_rn(f);
  *lo = f32_bits(f - bits_f32(*hi));
}

// hi = fp16(x), lo = fp16(x - hi) (3xFP16: 22 significant bits), from fp32(x)
// as the kernel's explicit-batch prologue does (x - hi is exact in fp32)
void f16_split(double xd, uint16_t* hi, uint16_t* lo) {
  const float x = (float)xd;
  *hi = f16_rne(x);
  const uint32_t hb = *hi;  // decode the half exactly
  const uint32_t ex = (hb >> 10) & 0x1Fu, man = hb & 0x3FFu;
  double hv = ex ? std::ldexp(1024.0 + man, (int)ex - 25) : std::ldexp((double)man, -24);
  if (hb & 0x8000u) hv = -hv;
  *lo = f16_rne(x - (float)hv);
}

// K-major, no-swizzle UMMA operand image of an N x K matrix (element (n,k) =
// B[k][n] of the fan_in x fan_out weight): core matrices 8 rows x 16 B,
// K-adjacent core matrices 128 B apart (LBO), 8-row groups SBO apart.
size_t pack_offset(uint32_t n, uint32_t k, uint32_t K, uint32_t esize) {
  const uint32_t kc = 16 / esize;
  const uint32_t sbo = (K / kc) * 128;
  return (size_t)(n / 8) * sbo + (size_t)(k / kc) * 128 + (n % 8) * 16 + (k % kc) * esize;
}

uint32_t make_idesc(int fmt, uint32_t N, uint32_t M) {
  // c_format F32 (bits 4-5 = 1), a/b format (bits 7-9, 10-12), K-major A and B,
  // n_dim = N >> 3 (bits 17-22), m_dim = M >> 4 (bits 24-28)
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool mul_ovf(uint64_t a, uint64_t b, uint64_t* out) { return __builtin_mul_overflow(a, b, out); }

// digits (group radix R, group 0 most significant) of delta mod prod(R)
void stride_digits(const uint32_t* R, uint64_t delta, uint32_t* dD) {
  for (int g = MAXG - 1; g >= 0; --g) {
    dD[g] = (uint32_t)(delta % R[g]);
    delta /= R[g];
  }
}

// ------------------------------------------------------------ kernel table
struct KernelInfo {
  const void* fn;
  int nslot, threads;
  bool bias_mma;
  bool a0_smem = false;  // SS-form A0 tiles + ones block in shared memory
  uint32_t red_bytes = 0;  // shared-memory partials of split-column epilogues
  bool pair = false;       // CTA-pair kernel (cluster of 2, cta_group::2, 256-row tiles)
  bool x_stage = false;    // predict rows staged in shared memory by bulk copies
  uint32_t a0_tiles = 1;   // shared-memory A0 tiles per slot (3xFP16: hi + lo)
  bool acc_stage = false;  // ensemble accumulator prefetched per tile into shared memory by bulk copies
  bool ens_pair = false;   // single-pass ensemble on CTA pairs (cluster of 2, 128-row tiles, members split)
  uint32_t w_mult = 1;     // member images resident per CTA (weight region = w_mult x w_bytes)
  uint32_t xch_bytes = 0;  // shared-memory exchange buffers (ensemble pairs)
  const void* fn_topk = nullptr;  // MODE_TOPK-only instantiation of fn (null: fn serves every mode)
};

template <int H, int SPG, int PREC>
KernelInfo kinfo_pair() {
  constexpr int NS = SURR_PAIR_NSUB;
  using C = CfgPair<H, NS>;
  KernelInfo ki{(const void*)&sweep_kernel_pair<H, SPG, NS, PREC>, 1, C::THREADS, true};
  ki.a0_smem = true;
  ki.red_bytes = (NS - 1) * TILE_M * 4;  // after the ones tile
  ki.pair = true;
  return ki;
}

template <int PREC, int H>
KernelInfo kinfo5() {
  using C = Cfg5<PREC, H>;
  KernelInfo ki{(const void*)&sweep_kernel5<PREC, H>, C::NSLOT, C::THREADS, false};
  ki.red_bytes = C::NSLOT * C::NSUB * TILE_M * 4;
  if (C::H16) {  // A0 hi / lo tiles in shared memory; partials after them
    ki.a0_smem = true;
    ki.a0_tiles = 2;
  }
  return ki;
}

template <int H>
KernelInfo kinfo6() {
  using C = Cfg6<H>;
  KernelInfo ki{(const void*)&sweep_kernel6<H>, C::NSLOT, C::THREADS, false};
  ki.a0_smem = true;  // A0 hi / lo tiles per slot
  ki.a0_tiles = 2;
  return ki;
}

template <int PREC, int H>
KernelInfo kinfo() {
  using C = Cfg<PREC, H>;
  return KernelInfo{(const void*)&sweep_kernel<PREC, H>, C::NSLOT, C::THREADS, C::BIAS_MMA};
}

template <int H, int SPG, int PREC, bool ENS = false>
KernelInfo kinfo3() {
  constexpr int NS = 4;  // four 128-row tiles in flight per SM
  using C = Cfg3<H, NS>;
  KernelInfo ki{(const void*)&sweep_kernel3<H, SPG, NS, PREC, ENS>, C::NSLOT, C::THREADS, true};
  ki.a0_smem = C::A0_SMEM;
  ki.x_stage = SPG == 0;  // the predict instantiation
  ki.acc_stage = ENS;
  return ki;
}

template <int H, int SPG, int PREC>
KernelInfo kinfo8() {
  // CB = 0 (all of half b in the L1 shadow, 64-column epilogue loads) measured
  // 1-2 % faster than CB = 16 (cfg2 3.49e10 vs 3.46e10, cfg5 3.15e10 vs 3.09e10
  // evals/s, same box); SURR_K8CB=16 selects the other split for A/B
  const char* v = getenv("SURR_K8CB");
  const bool cb16 = SPG != 0 && v && atoi(v) == 16;
  const void* fn = (const void*)&sweep_kernel8<H, SPG, PREC, 0>;
  if constexpr (SPG != 0)
    if (cb16) fn = (const void*)&sweep_kernel8<H, SPG, PREC, 16>;
  KernelInfo ki{fn, 4, 512, true};
  ki.x_stage = SPG == 0;  // the predict instantiation
  // the sweep's own instantiation (mode fixed to MODE_TOPK at compile time;
  // SURR_K8_ANYMODE=1 runs the any-mode kernel for A/B)
  const char* am = getenv("SURR_K8_ANYMODE");
  if constexpr (SPG != 0)
    if (!cb16 && !(am && atoi(am) == 1)) ki.fn_topk = (const void*)&sweep_kernel8<H, SPG, PREC, 0, MODE_TOPK>;
  ki.a0_smem = true;  // SS-form A0 tiles + the bias ones block in shared memory
  return ki;
}

template <int H, int SPG, int PREC, int GM>
KernelInfo kinfo8e() {
  KernelInfo ki{(const void*)&sweep_kernel8e<H, SPG, PREC, GM>, 4, 512, true};
  ki.a0_smem = true;
  ki.ens_pair = true;
  ki.w_mult = GM;
  ki.xch_bytes = 4 * 2 * TILE_M * 16;  // [slot][2 buffers][128 rows] x float4
  return ki;
}

// single-pass ensembles: 16-bit 14-128-128-1 members (device features folded),
// E = 4 or 8 (2 or 4 member images per CTA of the pair) (SURR_NO_ENS_PAIR=1: the multi-pass
// path, for A/B)
template <int PREC>
bool get_kernel_ens_pair16(uint32_t spg, uint32_t E, KernelInfo* ki) {
#define ENS_CASE(GM_)                                                     \
  if (E == 2 * GM_) {                                                     \
    *ki = spg == 4 ? kinfo8e<128, 4, PREC, GM_>() : kinfo8e<128, 2, PREC, GM_>(); \
    return true;                                                          \
  }
  ENS_CASE(2) ENS_CASE(4)
#undef ENS_CASE
  return false;
}
bool get_kernel_ens_pair(int prec, uint32_t H, uint32_t NL, uint32_t spg, uint32_t E, KernelInfo* ki) {
  const char* v = getenv("SURR_NO_ENS_PAIR");
  if ((v && atoi(v) == 1) || H != 128 || NL != 2 || (spg != 2 && spg != 4)) return false;
  if (prec == PREC_FP16) return get_kernel_ens_pair16<PREC_FP16>(spg, E, ki);
  if (prec == PREC_BF16) return get_kernel_ens_pair16<PREC_BF16>(spg, E, ki);
  return false;
}

bool uses_kernel3(int prec, uint32_t H, uint32_t NL) {
  return is16(prec) && NL <= 2 && (H == 32 || H == 64 || H == 128);
}
bool uses_quads(int prec, uint32_t H, uint32_t NL) {  // kernels with 4-parameter decoder groups
  return uses_kernel3(prec, H, NL) || (is16(prec) && H == 256);
}

template <int PREC>
bool get_kernel16(uint32_t H, uint32_t NL, KernelInfo* ki, uint32_t spg, bool ens) {
  // 16-bit nets whose weights exceed one SM (H = 256): CTA pairs
  if (H == 256) {
    *ki = spg == 4 ? kinfo_pair<256, 4, PREC>() : kinfo_pair<256, 2, PREC>();
    return true;
  }
  // nets with at most one hidden->hidden layer: four tiles in flight
  if (uses_kernel3(PREC, H, NL)) {
    // spg 0 = the predict instantiation
    if (H == 32) {
      *ki = spg == 4 ? kinfo3<32, 4, PREC>() : spg == 2 ? kinfo3<32, 2, PREC>() : kinfo3<32, 0, PREC>();
      return true;
    }
    if (H == 64) {
      *ki = spg == 4 ? kinfo3<64, 4, PREC>() : spg == 2 ? kinfo3<64, 2, PREC>() : kinfo3<64, 0, PREC>();
      return true;
    }
    if (H == 128) {
      // ensembles (cfg 4): the accumulator-staging instantiations of the quad-table and predict kernels
      if (ens && spg == 4) { *ki = kinfo3<128, 4, PREC, true>(); return true; }
      if (ens && spg == 0) { *ki = kinfo3<128, 0, PREC, true>(); return true; }
      // 14-128-128-1 sweeps: the final layer pipelined across tiles (SURR_K3=1:
      // sweep_kernel3 for same-box A/B)
      const char* k3 = getenv("SURR_K3");
      if (NL == 2 && !(k3 && atoi(k3) == 1)) {
        *ki = spg == 4 ? kinfo8<128, 4, PREC>() : spg == 2 ? kinfo8<128, 2, PREC>() : kinfo8<128, 0, PREC>();
        return true;
      }
      *ki = spg == 4 ? kinfo3<128, 4, PREC>() : spg == 2 ? kinfo3<128, 2, PREC>() : kinfo3<128, 0, PREC>();
      return true;
    }
  }
  return false;
}

bool get_kernel(int prec, uint32_t H, uint32_t NL, KernelInfo* ki, uint32_t spg = 2, bool ens = false) {
  if (prec == PREC_BF16 && get_kernel16<PREC_BF16>(H, NL, ki, spg, ens)) return true;
  if (prec == PREC_FP16 && get_kernel16<PREC_FP16>(H, NL, ki, spg, ens)) return true;
  // FP32 (3xTF32) nets with at most one hidden->hidden layer: self-issuing, split
  // columns, separate D2 region (measured faster than the general kernel; for
  // 1xTF32 the general two-slot kernel measured faster, 572 vs 482 TFLOP/s)
  // FP32 path as 3xFP16 with a hidden->hidden layer: three slots sharing the
  // last-layer region (SURR_VARIANT=9 selects the two-slot kernel for A/B runs)
  if (prec == PREC_FP32H && NL == 2) {
    const char* v = getenv("SURR_VARIANT");
    if (!(v && atoi(v) == 9)) {
      if (H == 32) { *ki = kinfo6<32>(); return true; }
      if (H == 64) { *ki = kinfo6<64>(); return true; }
      if (H == 128) { *ki = kinfo6<128>(); return true; }
    }
  }
  if (prec == PREC_FP32H || (prec == PREC_FP32 && NL <= 2)) {
#define CASE5(P_, H_) \
  if (prec == P_ && H == H_) { *ki = kinfo5<P_, H_>(); return true; }
    CASE5(PREC_FP32, 32) CASE5(PREC_FP32, 64) CASE5(PREC_FP32, 128)
    CASE5(PREC_FP32H, 32) CASE5(PREC_FP32H, 64) CASE5(PREC_FP32H, 128)
    CASE5(PREC_TF32, 32) CASE5(PREC_TF32, 64) CASE5(PREC_TF32, 128)
#undef CASE5
  }
#define CASE(P_, H_) \
  if (prec == P_ && H == H_) { *ki = kinfo<P_, H_>(); return true; }
  CASE(PREC_BF16, 32) CASE(PREC_BF16, 64) CASE(PREC_BF16, 128)
  CASE(PREC_FP16, 32) CASE(PREC_FP16, 64) CASE(PREC_FP16, 128)
  CASE(PREC_FP32, 32) CASE(PREC_FP32, 64) CASE(PREC_FP32, 128)
  CASE(PREC_TF32, 32) CASE(PREC_TF32, 64) CASE(PREC_TF32, 128)
#undef CASE
  return false;
}

surr_status check_device(surrogate* h, int dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return fail(h, SURR_E_NO_DEVICE, "no CUDA device");
  if (dev < 0 || dev >= n) return fail(h, SURR_E_NO_DEVICE, "device %d out of range (%d devices)", dev, n);
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0)
    return fail(h, SURR_E_NO_DEVICE, "device %d is sm_%d%d, this library is built for sm_100a", dev, prop.major,
                prop.minor);
  return SURR_OK;
}

// dynamic shared-memory layout of one K1 launch (offsets into p); returns bytes
size_t smem_layout(const KernelInfo& ki, KParams& p, uint32_t lut_bytes, uint32_t k, int mode) {
  const int nslot = ki.nslot;
  size_t off = align_up((size_t)p.w_bytes * ki.w_mult, 128);
  p.smem_lut = (uint32_t)off;
  off = align_up(off + (mode == MODE_PREDICT ? 0 : lut_bytes), 128);
  p.smem_lists = (uint32_t)off;
  off += (mode == MODE_TOPK ? 2ull * k * sizeof(surr_record) : 0);
  off = align_up(off, 128);
  p.smem_cand = (uint32_t)off;
  off += (mode == MODE_TOPK ? (size_t)nslot * 4 * CAND_CAP * sizeof(surr_record) : 0);  // last-sub warps
  off = align_up(off, 128);
  p.smem_misc = (uint32_t)off;
  off += 512;  // mbarriers [0 .. 31], TMEM slot address (+64), top-k scalars (+128), staging barriers (+256)
  p.smem_acc = (uint32_t)align_up(off, 128);
  off = p.smem_acc + (ki.acc_stage ? (size_t)nslot * 2 * TILE_M * 4 : 0);
  off = align_up(off, 1024);
  p.smem_a0 = (uint32_t)off;
  off += ki.a0_smem ? (size_t)nslot * ki.a0_tiles * 4096 : ki.red_bytes;
  p.smem_ones = (uint32_t)off;
  off += ki.a0_smem ? 4096 + ki.red_bytes : 0;
  off = align_up(off, 128);
  p.smem_x = (uint32_t)off;
  p.x_tile_bytes = TILE_M * p.P * 4;  // a multiple of 16 (bulk-copy granule)
  off += (mode == MODE_PREDICT && ki.x_stage) ? (size_t)nslot * p.x_tile_bytes : ki.xch_bytes;
  return off;
}
constexpr size_t SMEM_MAX = 227 * 1024;
// fused grid-merge tree: one ticket per node, TREE_NODES_PER_LEVEL per level, up to 9 levels (grid <= 256)
constexpr size_t CTR_BYTES = 9 * TREE_NODES_PER_LEVEL * sizeof(uint32_t);

// ------------------------------------------------------------ space / LUT
surr_status f16_range_check(surrogate* h, const std::vector<uint32_t>& radix, const std::vector<double>& values);
// k_hint: the top-k size the space is prepared for (shared-memory budget of the
// 4-parameter decoder table)
surr_status prepare_space(surrogate* h, const surr_space* sp, bool force, cudaStream_t st, uint32_t k_hint = 1) {
  if (!sp || !sp->radix || !sp->values) return fail(h, SURR_E_INVALID_ARG, "null space descriptor");
  const uint32_t P = sp->num_params;
  if (P == 0 || P > SURR_MAX_PARAMS) return fail(h, SURR_E_INVALID_ARG, "num_params %u out of range", P);
  if (P != h->P) return fail(h, SURR_E_INVALID_ARG, "space has %u params, model expects %u", P, h->P);
  uint64_t card = 1, nvals = 0;
  for (uint32_t j = 0; j < P; ++j) {
    if (sp->radix[j] == 0) return fail(h, SURR_E_INVALID_ARG, "radix[%u] == 0", j);
    if (mul_ovf(card, sp->radix[j], &card)) return fail(h, SURR_E_RANGE, "|S| does not fit in 64 bits");
    nvals += sp->radix[j];
  }
  std::vector<uint32_t> radix(sp->radix, sp->radix + P);
  std::vector<double> values(sp->values, sp->values + nvals);
  for (uint32_t j = 0, o = 0; j < P; o += radix[j], ++j)
    for (uint32_t d = 1; d < radix[j]; ++d)
      if (!(values[o + d] > values[o + d - 1]))
        return fail(h, SURR_E_INVALID_ARG, "value list %u not strictly increasing", j);
  const uint64_t end = sp->end ? sp->end : card;
  if (sp->begin > end || end > card)
    return fail(h, SURR_E_INVALID_ARG, "bad range [%llu, %llu) of |S| = %llu", (unsigned long long)sp->begin,
                (unsigned long long)end, (unsigned long long)card);
  auto table_entries = [&](uint32_t spg_) {
    uint64_t e = 0;
    for (uint32_t g = 0; g < (uint32_t)K0 / spg_; ++g) {
      uint64_t r = 1;
      for (uint32_t q = 0; q < spg_; ++q) r *= (spg_ * g + q) < P ? radix[spg_ * g + q] : 1u;
      e += r;
    }
    return e;
  };
  // quadruples when the kernel takes them and a top-k launch still fits in
  // shared memory with the larger table (e.g. the paper's 10/12-value lists:
  // 2 x 14,400 + 2 x 120 + ... entries, 117 KB next to cfg2's 36 KB of weights)
  uint32_t spg = 2;
  if (uses_quads(h->prec, h->H, h->NL) && table_entries(4) * 8 <= 120 * 1024) {
    KernelInfo ki4;
    KParams tmp = h->mp;
    if (get_kernel(h->prec, h->H, h->NL, &ki4, 4, h->members.size() > 1) &&
        smem_layout(ki4, tmp, (uint32_t)align_up(table_entries(4) * 8, 16), std::max(k_hint, 1u), MODE_TOPK) <=
            SMEM_MAX)
      spg = 4;
  }
  if (!force && h->space_valid && radix == h->c_radix && values == h->c_values && spg == h->spg) {
    h->sp.begin = sp->begin;
    h->sp.end = end;
    h->card = card;
    return SURR_OK;
  }
  // the cached space is replaced: nothing of it stays valid if a check below fails
  h->space_valid = false;
  if (f16_range_check(h, radix, values) != SURR_OK) return SURR_E_RANGE;

  // super digits: group g holds A0 slots [spg g, spg (g+1)) (parameter j in slot j,
  // the ones slot P carrying b_1, zeros after); R_g = product of its parameters'
  // radices.  spg = 4: 8-byte entries = four packed bf16 columns (BF16 kernels
  // with quadruple groups, see above), else 2.
  const bool bf = is16(h->prec);
  const bool h3 = h->prec == PREC_FP32H;  // 3xFP16: fp16 hi pair + fp16 lo pair per entry
  KParams k = h->sp;  // committed to the handle only once the table is uploaded
  k.begin = sp->begin;
  k.end = end;
  std::vector<uint32_t> voff(P);
  for (uint32_t j = 0, o = 0; j < P; o += radix[j], ++j) voff[j] = o;
  // StandardScaler / min-max affine map z = (x - shift) / scale, evaluated as the
  // kernels' explicit-batch prologue does: one fp32 FMA fma(fp32(x), fp32(1/scale),
  // fp32(-shift/scale)) (|dz| ~ 1e-7 |z| against the exact map)
  auto slot_val = [&](uint32_t slot, uint32_t d) -> double {
    if (slot < P) return (double)std::fmaf((float)values[voff[slot] + d], h->mp.zinv[slot], h->mp.zc[slot]);
    return slot == P ? 1.0 : 0.0;
  };
  const uint32_t ng = K0 / spg;
  // bf16 / fp16: spg packed halves; 3xFP16 (spg 2): fp16 hi pair + lo pair; tf32 (spg 2): hi pair + lo pair
  const size_t esz = bf ? 2 * spg : h3 ? 8 : 16;
  size_t entries = 0;
  for (uint32_t g = 0; g < (uint32_t)MAXG; ++g) {
    uint64_t r = 1;
    if (g < ng)
      for (uint32_t q = 0; q < spg; ++q) r *= (spg * g + q) < P ? radix[spg * g + q] : 1u;
    k.R[g] = (uint32_t)r;
    k.lut_off[g] = (uint32_t)entries;
    entries += g < ng ? r : 0;
  }
  if (entries * esz > 120 * 1024) return fail(h, SURR_E_UNSUPPORTED, "value table too large (%zu entries)", entries);
  std::vector<uint8_t> lut(align_up(entries * esz, 16), 0);
  for (uint32_t g = 0; g < ng; ++g) {
    for (uint32_t D = 0; D < k.R[g]; ++D) {
      // digits of the group's slots, first slot most significant
      uint32_t dig[4] = {0, 0, 0, 0}, rem = D;
      for (int q = (int)spg - 1; q >= 0; --q) {
        const uint32_t slot = spg * g + q;
        const uint32_t r = slot < P ? radix[slot] : 1u;
        dig[q] = rem % r;
        rem /= r;
      }
      uint8_t* e = lut.data() + (k.lut_off[g] + (size_t)D) * esz;
      if (bf) {
        for (uint32_t q = 0; q < spg; ++q) {
          const uint16_t v = h16_rne(h->prec, (float)slot_val(spg * g + q, dig[q]));
          memcpy(e + 2 * q, &v, 2);
        }
      } else if (h3) {
        uint16_t w[4];
        f16_split(slot_val(2 * g, dig[0]), &w[0], &w[2]);
        f16_split(slot_val(2 * g + 1, dig[1]), &w[1], &w[3]);
        memcpy(e, w, 8);
      } else {
        uint32_t w[4];
        tf32_split(slot_val(2 * g, dig[0]), &w[0], &w[2]);
        tf32_split(slot_val(2 * g + 1, dig[1]), &w[1], &w[3]);
        memcpy(e, w, 16);
      }
    }
  }
  // stream-ordered upload into the ring's other slot: sweeps queued earlier (on
  // any stream) keep reading the slot their launch captured
  void* dl = nullptr;
  surr_status urc = ring_upload(h, h->lring, lut.data(), lut.size(), st, false, &dl);
  if (urc) return urc;
  k.lut_gmem = dl;
  k.lut_bytes = (uint32_t)lut.size();
  h->sp = k;
  h->card = card;
  h->lut.swap(lut);
  h->c_radix = radix;
  h->c_values = values;
  h->spg = spg;
  h->space_valid = true;
  return SURR_OK;
}

// FP16 operands overflow above 65504.  Interval bound of every activation that
// becomes a UMMA operand (z, and h_l = relu(W_l h_{l-1} + b_l) for l < NL) over
// the space's value lists; SURR_E_RANGE if one can reach the FP16 limit.
surr_status f16_range_check(surrogate* h, const std::vector<uint32_t>& radix, const std::vector<double>& values) {
  if (h->prec != PREC_FP16 && h->prec != PREC_FP32H) return SURR_OK;
  const uint32_t P = h->P, H = h->H;
  const double LIM = 65504.0 * (1.0 - 1.0 / 2048.0);
  std::vector<double> zlo(K0, 0.0), zhi(K0, 0.0);
  for (uint32_t j = 0, o = 0; j < P; o += radix[j], ++j) {
    const double a = (values[o] - h->hshift[j]) / h->hscale[j];
    const double b = (values[o + radix[j] - 1] - h->hshift[j]) / h->hscale[j];  // lists increase
    zlo[j] = std::min(a, b);
    zhi[j] = std::max(a, b);
    if (std::max(std::fabs(a), std::fabs(b)) >= LIM)
      return fail(h, SURR_E_RANGE, "normalised parameter %u reaches %g: outside the FP16 range", j,
                  std::max(std::fabs(a), std::fabs(b)));
  }
  zlo[P] = zhi[P] = 1.0;  // ones slot (b_1)
  double worst = 0.0;
  for (size_t e = 0; e < h->rb_B1.size(); ++e) {
    const std::vector<double>& B1 = h->rb_B1[e];
    std::vector<double> U(H);
    for (uint32_t n = 0; n < H; ++n) {
      double u = 0.0;
      for (uint32_t j = 0; j <= P; ++j) u += std::max(B1[(size_t)j * H + n] * zlo[j], B1[(size_t)j * H + n] * zhi[j]);
      U[n] = std::max(0.0, u);
    }
    if (h->NL >= 2) worst = std::max(worst, *std::max_element(U.begin(), U.end()));
    for (size_t l = 0; l < h->rb_W[e].size(); ++l) {
      const std::vector<double>& W = h->rb_W[e][l];
      std::vector<double> V(H);
      for (uint32_t m = 0; m < H; ++m) {
        double u = h->rb_b[e][l][m];
        for (uint32_t n = 0; n < H; ++n) u += std::max(0.0, W[(size_t)n * H + m]) * U[n];
        V[m] = std::max(0.0, u);
      }
      U.swap(V);
      worst = std::max(worst, *std::max_element(U.begin(), U.end()));
    }
  }
  if (worst >= LIM)
    return fail(h, SURR_E_RANGE,
                "hidden activations can reach %g over this space: outside the FP16 range (use BF16 or "
                "SURR_PREC_FP32_3XTF32)", worst);
  return SURR_OK;
}

struct Launch {
  KernelInfo ki;
  int grid;
  size_t smem;
  KParams p;
};

surr_status plan(surrogate* h, uint64_t begin, uint64_t end, uint32_t k, int mode, Launch* L, uint32_t member = 0,
                 const KernelInfo* force = nullptr) {
  if (force) L->ki = *force;
  else if (!get_kernel(h->prec, h->H, h->NL, &L->ki, mode == MODE_PREDICT ? 0 : h->spg, h->members.size() > 1))
    return fail(h, SURR_E_UNSUPPORTED, "no kernel for H=%u", h->H);
  KParams p = h->members.empty() ? h->mp : h->members[member];
  if (L->ki.ens_pair) {  // all members in one launch: member 0's image is the base of all of them
    const uint32_t E = (uint32_t)h->members.size();
    p.ens_gm = L->ki.w_mult;
    p.ens_e = E;
    for (uint32_t e = 0; e < E && e < 16; ++e) p.ens_c[e] = h->members[e].c_out;
    for (uint32_t e = 0; e < E && e < 8; ++e) memcpy(p.ens_w[e], h->members[e].fin_w, sizeof p.ens_w[e]);
    p.inv_e = 1.0f / (float)E;
  }
  const KParams& s = h->sp;
  if (mode != MODE_PREDICT) {
    memcpy(p.R, s.R, sizeof p.R);
    memcpy(p.lut_off, s.lut_off, sizeof p.lut_off);
    p.lut_gmem = s.lut_gmem;
    p.lut_bytes = s.lut_bytes;
  } else {
    for (int g = 0; g < MAXG; ++g) { p.R[g] = 1; p.lut_off[g] = 0; p.dD[g] = 0; }
    p.lut_bytes = 0;
  }
  p.begin = begin;
  p.end = end;
  const uint64_t rows_per_tile = L->ki.pair ? 2 * TILE_M : TILE_M;
  p.num_tiles = (end - begin + rows_per_tile - 1) / rows_per_tile;
  const int nslot = L->ki.nslot;
  uint64_t want = (p.num_tiles + nslot - 1) / nslot;
  if (L->ki.pair) {  // clusters of two CTAs, one 256-row tile per pair at a time
    L->grid = 2 * (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)h->sms / 2, p.num_tiles));
  } else if (L->ki.ens_pair) {  // clusters of two CTAs sweeping the same tiles (members split)
    L->grid = 2 * (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)h->sms / 2, want));
  } else {
    L->grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)h->sms, want));
  }
  p.dTiles = (uint32_t)(nslot * (L->ki.ens_pair ? L->grid / 2 : L->grid));
  if (mode != MODE_PREDICT) stride_digits(p.R, (uint64_t)p.dTiles * TILE_M, p.dD);
  p.k = mode == MODE_TOPK ? k : 1;
  L->smem = smem_layout(L->ki, p, p.lut_bytes, k, mode);
  if (L->smem > SMEM_MAX) return fail(h, SURR_E_UNSUPPORTED, "shared memory %zu B exceeds 227 KB", L->smem);
  L->p = p;
  return SURR_OK;
}

surr_status launch(surrogate* h, Launch& L, int mode, cudaStream_t st) {
  const void* fn = (mode == MODE_TOPK && L.ki.fn_topk) ? L.ki.fn_topk : L.ki.fn;
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->timing) {  // every K1 launch (ensembles run one per member)
    if (h->ev_used + 2 > h->ev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        h->ev.push_back(e);
      }
    }
    e0 = h->ev[h->ev_used];
    e1 = h->ev[h->ev_used + 1];
    h->ev_used += 2;
    CU(cudaEventRecord(e0, st));
  }
  void* args[] = {(void*)&L.p, (void*)&mode};
  if (L.ki.pair || L.ki.ens_pair) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(L.ki.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelExC(&cfg, fn, args));
  } else {
    CU(cudaLaunchKernel(fn, dim3(L.grid), dim3(L.ki.threads), args, L.smem, st));
  }
  if (e1) CU(cudaEventRecord(e1, st));
  ++h->launches;
  // the launch reads the weight image and (sweeps) the value table by pointer
  surr_status rc = ring_mark_use(h, h->wring, st);
  if (!rc && mode != MODE_PREDICT) rc = ring_mark_use(h, h->lring, st);
  return rc;
}

surr_status ensure_recs(surrogate* h, size_t n) {
  if (n <= h->d_recs_cap) return SURR_OK;
  if (h->d_recs) cudaFree(h->d_recs);
  h->d_recs = nullptr;
  if (cudaMalloc(&h->d_recs, n * sizeof(surr_record)) != cudaSuccess) return fail(h, SURR_E_OOM, "cudaMalloc recs");
  h->d_recs_cap = n;
  return SURR_OK;
}

surr_status launch_merge(surrogate* h, const surr_record* in, uint32_t lists, uint32_t k_in, uint32_t k,
                         uint64_t* oi, float* ot, surr_record* orec, cudaStream_t st) {
  const size_t budget = 200 * 1024 - 2ull * k * sizeof(surr_record);
  const uint32_t slot = std::max(k_in, k);  // list slot stride in shared memory (merge_kernel)
  uint32_t chunk = (uint32_t)std::max<size_t>(1, budget / (2ull * slot * sizeof(surr_record)));
  chunk = std::min<uint32_t>(chunk, std::max<uint32_t>(lists, 1));
  const size_t smem = (2ull * k + 2ull * chunk * slot) * sizeof(surr_record);
  if (smem > 227 * 1024) return fail(h, SURR_E_UNSUPPORTED, "merge needs %zu B shared memory", smem);
  CU(cudaFuncSetAttribute((const void*)merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  merge_kernel<<<1, 1024, smem, st>>>(in, lists, k_in, k, chunk, oi, ot, orec);
  CU(cudaGetLastError());
  ++h->launches;
  return SURR_OK;
}

// K1 over [begin, end) in `mode`, with the ensemble passes when E > 1: per
// chunk of <= 2^28 configs, members 0..E-2 accumulate t into d_acc and the last
// member averages and emits (top-k records at recs + lists * k, or dense t,
// or predict rows).  Returns the number of record lists written.
// Merged top-k outputs of a sweep; K1 merges its own lists (a9: a binary tree of CTAs) when
// the sweep is a single top-k launch whose shared memory holds the merge.
struct MergeOut {
  uint64_t* idx;
  float* t;
  surr_record* recs;
  bool fused = false;  // out: K1 wrote the merged outputs
};

surr_status run_k1(surrogate* h, uint64_t begin, uint64_t end, uint32_t k, int mode, float* t_dense, const float* x,
                   cudaStream_t st, uint32_t* lists_out, MergeOut* mo = nullptr) {
  const uint32_t E = (uint32_t)std::max<size_t>(1, h->members.size());
  // ensembles: one pass on CTA pairs when the members fit (no accumulator, one launch)
  if (E > 1 && mode != MODE_PREDICT) {
    KernelInfo kp;
    Launch L;
    if (get_kernel_ens_pair(h->prec, h->H, h->NL, h->spg, E, &kp) &&
        plan(h, begin, end, k, mode, &L, 0, &kp) == SURR_OK) {
      if (mode == MODE_TOPK) {
        surr_status rc = ensure_recs(h, (size_t)L.grid * k);
        if (rc) return rc;
      }
      L.p.recs = h->d_recs;
      L.p.t_dense = t_dense;
      L.p.a0_dump = h->a0_dump;
      L.p.a0_stride = h->a0_stride;
      L.p.trace = h->trace;
      L.p.trace_n = h->trace_n;
      const size_t need1 = 3ull * k * sizeof(surr_record);  // the merge tree's two lists + result
      const bool fuse = mo && mode == MODE_TOPK && L.smem >= need1 && L.grid <= (int)TREE_NODES_PER_LEVEL &&
                        !getenv("SURR_NO_FUSED_MERGE");
      if (fuse) {
        L.p.done_ctr = h->d_ctr;
        L.p.out_idx = mo->idx;
        L.p.out_t = mo->t;
        L.p.out_recs = mo->recs;
      }
      if (mo) mo->fused = fuse;
      surr_status rc = launch(h, L, mode, st);
      if (rc) return rc;
      *lists_out = (uint32_t)L.grid;
      return SURR_OK;
    }
    h->err.clear();  // not applicable (shape, E, or shared memory): the multi-pass path below
  }
  const uint64_t chunk = E == 1 ? (end - begin) : (1ull << 28);
  // record lists of every chunk's final pass
  uint64_t lists = 0, nchunks = 0;
  uint32_t fuse_chunk = 0;  // 1: K1 can merge its grid's lists itself (a9 tree), 0: K2 merges
  for (uint64_t c0 = begin; c0 < end; c0 += chunk) {
    Launch L;
    surr_status rc = plan(h, c0, std::min(end, c0 + chunk), k, mode, &L);
    if (rc) return rc;
    lists += (uint64_t)L.grid;
    ++nchunks;
    const size_t need1 = 3ull * k * sizeof(surr_record);  // the merge tree's two lists + result
    if (L.smem >= need1 && L.grid <= (int)TREE_NODES_PER_LEVEL) fuse_chunk = 1;
  }
  const bool fuse = mo && mode == MODE_TOPK && nchunks == 1 && fuse_chunk >= 1 && !getenv("SURR_NO_FUSED_MERGE");
  if (mo) mo->fused = fuse;
  if (mode == MODE_TOPK) {
    surr_status rc = ensure_recs(h, (size_t)lists * k);
    if (rc) return rc;
  }
  if (E > 1) {
    const size_t need = (size_t)std::min<uint64_t>(chunk, end - begin);
    if (need > h->d_acc_cap) {
      cudaFree(h->d_acc);
      h->d_acc = nullptr;
      if (cudaMalloc(&h->d_acc, need * sizeof(float)) != cudaSuccess) return fail(h, SURR_E_OOM, "cudaMalloc acc");
      h->d_acc_cap = need;
    }
  }
  uint64_t done = 0;
  for (uint64_t c0 = begin; c0 < end; c0 += chunk) {
    const uint64_t c1 = std::min(end, c0 + chunk);
    int grid = 0;
    for (uint32_t e = 0; e < E; ++e) {
      const bool last = e + 1 == E;
      const int m = mode == MODE_PREDICT ? MODE_PREDICT : (last ? mode : MODE_DENSE);
      Launch L;
      surr_status rc = plan(h, c0, c1, k, m, &L, e);
      if (rc) return rc;
      grid = L.grid;
      if (E > 1) {
        L.p.acc_mode = e == 0 ? 1u : (last ? 3u : 2u);
        L.p.t_acc = h->d_acc;
        L.p.acc_base = c0;
        L.p.inv_e = 1.0f / (float)E;
        // members >= 1 read t_acc[I - c0]: tile-aligned, so 512-byte bulk copies per tile
        L.p.acc_tma = (L.ki.acc_stage && e > 0 && ((uintptr_t)h->d_acc % 16) == 0) ? 1u : 0u;
      }
      L.p.recs = h->d_recs + done * k;
      if (fuse && last) {
        L.p.done_ctr = h->d_ctr;
        L.p.out_idx = mo->idx;
        L.p.out_t = mo->t;
        L.p.out_recs = mo->recs;
      }
      L.p.t_dense = t_dense ? t_dense + (c0 - begin) : nullptr;
      L.p.x = x;
      L.p.a0_dump = h->a0_dump;
      L.p.a0_stride = h->a0_stride;
      // bulk copies need 16-byte aligned rows blocks: x itself, and c0 P 4 bytes
      L.p.x_tma = (L.ki.x_stage && x && ((uintptr_t)x % 16) == 0 && (c0 * L.p.P * 4) % 16 == 0) ? 1u : 0u;
      L.p.trace = h->trace;
      L.p.trace_n = h->trace_n;
      { const char* v = getenv("SURR_VARIANT"); L.p.variant = v ? (uint32_t)atoi(v) : 0u; }
      if (L.p.variant == 4) L.p.acc_tma = 0;  // A/B: accumulator read at use
      rc = launch(h, L, m, st);
      if (rc) return rc;
    }
    done += (uint64_t)grid;
  }
  *lists_out = (uint32_t)done;
  return SURR_OK;
}

surr_status sweep_common(surrogate* h, const surr_space* space, uint32_t k, uint64_t* idx_dev, float* t_dev,
                         surr_record* recs_dev, uint32_t* count_host, cudaStream_t st, bool force) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!h->loaded) return fail(h, SURR_E_NOT_LOADED, "no model loaded");
  if (k == 0 || k > SURR_K_MAX) return fail(h, SURR_E_INVALID_ARG, "k = %u outside 1..%u", k, SURR_K_MAX);
  CU(cudaSetDevice(h->dev));
  surr_status rc = prepare_space(h, space, force, st, k);
  if (rc) return rc;
  const uint64_t begin = h->sp.begin, end = h->sp.end;
  const uint64_t n = end - begin;
  if (count_host) *count_host = (uint32_t)std::min<uint64_t>(k, n);
  h->launches = 0;
  if (n == 0) {
    // empty range: all-sentinel result through the merge kernel (zero lists)
    return launch_merge(h, h->d_recs, 0, k, k, idx_dev, t_dev, recs_dev, st);
  }
  uint32_t lists = 0;
  MergeOut mo{idx_dev, t_dev, recs_dev};
  rc = run_k1(h, begin, end, k, MODE_TOPK, nullptr, nullptr, st, &lists, &mo);
  if (rc) return rc;
  if (mo.fused) return SURR_OK;  // K1 merged its grid's lists (a9 tree): one kernel per sweep
  return launch_merge(h, h->d_recs, lists, k, k, idx_dev, t_dev, recs_dev, st);
}

}  // namespace

// ================================================================== C ABI
extern "C" {

surr_status surrogate_create(int cuda_device, surrogate_t** out) {
  if (!out) return fail(nullptr, SURR_E_INVALID_ARG, "null out");
  *out = nullptr;
  surrogate* h = nullptr;
  surr_status rc = check_device(nullptr, cuda_device);
  if (rc) return rc;
  h = new surrogate();
  h->dev = cuda_device;
  if (cudaSetDevice(cuda_device) != cudaSuccess) { delete h; return fail(nullptr, SURR_E_CUDA, "cudaSetDevice"); }
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, cuda_device);
  if (cudaMalloc(&h->d_merged, SURR_K_MAX * sizeof(surr_record)) != cudaSuccess ||
      cudaMalloc(&h->d_ctr, CTR_BYTES) != cudaSuccess || cudaMemset(h->d_ctr, 0, CTR_BYTES) != cudaSuccess) {
    cudaFree(h->d_merged);
    delete h;
    return fail(nullptr, SURR_E_OOM, "cudaMalloc");
  }
  *out = h;
  return SURR_OK;
}

void surrogate_destroy(surrogate_t* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  ring_free(h->wring);
  ring_free(h->lring);
  cudaFree(h->d_recs); cudaFree(h->d_merged); cudaFree(h->d_ctr);
  cudaFree(h->d_acc);
  for (auto e : h->ev) cudaEventDestroy(e);
  delete h;
}

const char* surrogate_last_error(const surrogate_t* h) { return h ? h->err.c_str() : g_err.c_str(); }

uint32_t surrogate_last_launches(const surrogate_t* h) { return h ? h->launches : 0; }

surr_status surrogate_arith(const surrogate_t* h, uint32_t* mma_kind, uint32_t* passes, double* issued_flops) {
  if (!h || !mma_kind || !passes || !issued_flops) return SURR_E_INVALID_ARG;
  if (!h->loaded) return SURR_E_NOT_LOADED;
  KernelInfo ki;
  if (!get_kernel(h->prec, h->H, h->NL, &ki)) return SURR_E_UNSUPPORTED;
  const bool k16 = is16(h->prec) || h->prec == PREC_FP32H;
  const bool split = h->prec == PREC_FP32 || h->prec == PREC_FP32H;
  *mma_kind = k16 ? 0u : 1u;
  *passes = split ? 3u : 1u;
  const double H = h->H;
  const double p1 = is16(h->prec) ? 1.0 : 3.0;                // layer 1 (K0 = 16)
  const double kb = k16 ? 16.0 : 8.0;                         // bias K block
  const double pb = split ? (k16 ? 1.0 : 2.0) : 1.0;
  const double hidden = H * H * (*passes) + (ki.bias_mma ? kb * H * pb : 0.0);
  *issued_flops = 2.0 * (K0 * H * p1 + (double)(h->NL - 1) * hidden);
  return SURR_OK;
}

uint32_t surrogate_table_bytes(const surrogate_t* h) { return h && h->space_valid ? h->sp.lut_bytes : 0; }

surr_status surrogate_space_size(const surr_space* sp, uint64_t* out) {
  surrogate* h = nullptr;
  if (!sp || !out || !sp->radix) return fail(h, SURR_E_INVALID_ARG, "null argument");
  if (sp->num_params == 0 || sp->num_params > SURR_MAX_PARAMS) return fail(h, SURR_E_INVALID_ARG, "num_params");
  uint64_t c = 1;
  for (uint32_t j = 0; j < sp->num_params; ++j) {
    if (sp->radix[j] == 0) return fail(h, SURR_E_INVALID_ARG, "radix[%u] == 0", j);
    if (mul_ovf(c, sp->radix[j], &c)) return fail(h, SURR_E_RANGE, "|S| does not fit in 64 bits");
  }
  *out = c;
  return SURR_OK;
}

surr_status surrogate_load_weights(surrogate_t* h, const surr_model* m) {
  if (!h || !m || !m->widths || !m->W || !m->b || !m->x_shift || !m->x_scale)
    return fail(h, SURR_E_INVALID_ARG, "null argument");
  const uint32_t L = m->num_layers;
  if (L < 2 || L - 1 > SURR_MAX_HIDDEN_LAYERS)
    return fail(h, SURR_E_UNSUPPORTED, "num_layers %u: need 1..%u hidden layers", L, SURR_MAX_HIDDEN_LAYERS);
  if (m->ensemble < 1 || m->ensemble > 64) return fail(h, SURR_E_INVALID_ARG, "ensemble %u outside 1..64", m->ensemble);
  const uint32_t E = m->ensemble;
  if (m->precision != SURR_PREC_BF16 && m->precision != SURR_PREC_FP32 && m->precision != SURR_PREC_TF32 &&
      m->precision != SURR_PREC_FP16 && m->precision != SURR_PREC_FP32_3XTF32)
    return fail(h, SURR_E_INVALID_ARG, "precision %d", (int)m->precision);
  const bool p16 = m->precision == SURR_PREC_BF16 || m->precision == SURR_PREC_FP16;
  const uint32_t F = m->widths[0], H = m->widths[1];
  if (m->widths[L] != 1) return fail(h, SURR_E_INVALID_ARG, "output width must be 1");
  for (uint32_t l = 1; l < L; ++l)
    if (m->widths[l] != H) return fail(h, SURR_E_UNSUPPORTED, "hidden widths must be equal");
  if (H != 32 && H != 64 && H != 128 && !(H == 256 && p16))
    return fail(h, SURR_E_UNSUPPORTED, "hidden width %u not in {32,64,128} (256: BF16 / FP16 only)", H);
  if (m->num_const_features > F || (m->num_const_features && !m->const_features))
    return fail(h, SURR_E_INVALID_ARG, "const features");
  const uint32_t P = F - m->num_const_features;
  if (P == 0 || P + 1 > (uint32_t)K0) return fail(h, SURR_E_UNSUPPORTED, "%u tuning parameters: need 1..15", P);
  for (uint32_t l = 0; l < E * L; ++l)
    if (!m->W[l] || !m->b[l]) return fail(h, SURR_E_INVALID_ARG, "null layer %u", l);
  // non-finite parameters (e.g. a diverged fit) would make every prediction NaN
  for (uint32_t e = 0; e < E; ++e)
    for (uint32_t l = 0; l < L; ++l) {
      const size_t nw = (size_t)m->widths[l] * m->widths[l + 1];
      for (size_t i = 0; i < nw; ++i)
        if (!std::isfinite(m->W[e * L + l][i]))
          return fail(h, SURR_E_INVALID_ARG, "member %u layer %u: non-finite weight at %zu", e, l, i);
      for (uint32_t i = 0; i < m->widths[l + 1]; ++i)
        if (!std::isfinite(m->b[e * L + l][i]))
          return fail(h, SURR_E_INVALID_ARG, "member %u layer %u: non-finite bias at %u", e, l, i);
    }
  for (uint32_t j = 0; j < F; ++j)
    if (!std::isfinite(m->x_shift[j]) || !std::isfinite(m->x_scale[j]))
      return fail(h, SURR_E_INVALID_ARG, "non-finite input scaler at %u", j);
  if (!std::isfinite(m->y_mean) || !std::isfinite(m->y_scale))
    return fail(h, SURR_E_INVALID_ARG, "non-finite target scaler");
  CU(cudaSetDevice(h->dev));

  // the FP32 path runs as 3xFP16 where its kernels exist (H <= 128: twice the
  // tensor rate of 3xTF32, the same 22 significant bits), else (or when forced)
  // as 3xTF32
  const int prec = m->precision == SURR_PREC_BF16   ? PREC_BF16
                   : m->precision == SURR_PREC_FP16 ? PREC_FP16
                   : m->precision == SURR_PREC_TF32 ? PREC_TF32
                   : m->precision == SURR_PREC_FP32 && H <= 128 ? PREC_FP32H
                                                    : PREC_FP32;
  const uint32_t NL = L - 1;
  std::vector<double> shift(F), scale(F);
  for (uint32_t j = 0; j < F; ++j) {
    shift[j] = m->x_shift[j];
    scale[j] = m->x_scale[j] == 0.0 ? 1.0 : m->x_scale[j];
  }
  std::vector<KParams> mps(E);
  std::vector<std::vector<uint8_t>> imgs(E);
  std::vector<std::vector<double>> rb_B1(E);
  std::vector<std::vector<std::vector<double>>> rb_W(E), rb_b(E);
  for (uint32_t e = 0; e < E; ++e) {
    // layer 1 operand rows: z_0..z_{P-1}, ones slot carrying b_1 + W1[const] z_const, zeros
    const double* W1 = m->W[e * L + 0];
    std::vector<double> B1((size_t)K0 * H, 0.0);  // [k][n]
    for (uint32_t kk = 0; kk < P; ++kk)
      for (uint32_t n = 0; n < H; ++n) B1[(size_t)kk * H + n] = W1[(size_t)kk * H + n];
    for (uint32_t n = 0; n < H; ++n) {
      double b = m->b[e * L + 0][n];
      for (uint32_t c = 0; c < m->num_const_features; ++c) {
        const double zc = (m->const_features[c] - shift[P + c]) / scale[P + c];
        b += W1[(size_t)(P + c) * H + n] * zc;
      }
      B1[(size_t)P * H + n] = b;
    }
    rb_B1[e] = B1;
    for (uint32_t l = 1; l + 1 < NL; ++l) {  // hidden->hidden layers feeding another UMMA
      rb_W[e].emplace_back(m->W[e * L + l], m->W[e * L + l] + (size_t)H * H);
      rb_b[e].emplace_back(m->b[e * L + l], m->b[e * L + l] + H);
    }
    if (prec == PREC_FP16 || prec == PREC_FP32H) {
      double wmax = 0.0;
      for (double x : B1) wmax = std::max(wmax, std::fabs(x));
      for (uint32_t l = 1; l < NL; ++l)
        for (size_t i = 0; i < (size_t)H * H; ++i) wmax = std::max(wmax, std::fabs(m->W[e * L + l][i]));
      for (uint32_t l = 1; l < NL; ++l)
        for (uint32_t i = 0; i < H; ++i) wmax = std::max(wmax, std::fabs(m->b[e * L + l][i]));
      if (wmax >= 65504.0 * (1.0 - 1.0 / 2048.0))
        return fail(h, SURR_E_RANGE, "weight magnitude %g outside the FP16 range", wmax);
    }
    const bool bf = is16(prec) || prec == PREC_FP32H;  // 16-bit operand image
    const uint32_t esz = bf ? 2 : 4;
    KernelInfo ki;
    if (!get_kernel(prec, H, L - 1, &ki)) return fail(h, SURR_E_UNSUPPORTED, "no kernel for H=%u", H);
    const bool bias_mma = ki.bias_mma;     // hidden biases as an extra UMMA K block
    const uint32_t kstep = bf ? 16 : 8;
    const uint32_t KH = H + (bias_mma ? kstep : 0);  // K extent of a hidden-layer B image
    const bool lo1 = !is16(prec);          // layer 1 carries a lo part (TF32 modes, 3xFP16)
    const bool loh = prec == PREC_FP32 || prec == PREC_FP32H;  // hidden layers carry a lo part
    // CTA-pair kernel: rank r's image holds B columns [r NR, (r+1) NR) of every layer
    const uint32_t ranks = ki.pair ? 2 : 1;
    const uint32_t NR = H / ranks;
    const size_t b1_bytes = (size_t)NR * K0 * esz;
    const size_t bh_bytes = (size_t)NR * KH * esz;
    KParams p{};
    size_t off = 0;
    p.off_b1 = (uint32_t)off; off += b1_bytes;
    p.off_b1lo = lo1 ? (uint32_t)off : p.off_b1; off += lo1 ? b1_bytes : 0;
    off = align_up(off, 128);
    p.off_bh = (uint32_t)off;
    p.lo_delta_h = (uint32_t)bh_bytes;
    p.stride_bh = (uint32_t)align_up(bh_bytes * (loh ? 2 : 1), 128);
    off += (size_t)(NL - 1) * p.stride_bh;
    off = align_up(off, 16);
    p.off_fin = (uint32_t)off;  // final-layer [w' (H floats), -b (H floats)] for shared-memory readers
    off += 2ull * H * 4;
    p.w_bytes = (uint32_t)align_up(std::max<size_t>(off, 128), 128);
    {  // refuse at load time a net whose weight image cannot fit next to the smallest launch
      KParams probe = p;
      probe.P = P;
      if (smem_layout(ki, probe, 0, 1, MODE_DENSE) > SMEM_MAX)
        return fail(h, SURR_E_UNSUPPORTED, "weights of this net (%u B in the precision's operand format) do not fit "
                    "shared memory", p.w_bytes);
    }
    p.w_rank_stride = p.w_bytes;
    std::vector<uint8_t> img((size_t)p.w_bytes * ranks, 0);

    // image row n of rank r <- output column gcol(r, n).  Single CTA: n.  CTA
    // pair (N-half UMMAs of N = H/2, each CTA supplying H/4 B rows): rank r's
    // rows [h H/4, (h+1) H/4) are columns h H/2 + r H/4 + [0, H/4) of half h
    auto gcol = [&](uint32_t r, uint32_t n) -> uint32_t {
      if (ranks == 1) return n;
      const uint32_t Q = H / 4;
      return (n / Q) * (H / 2) + r * Q + n % Q;
    };
    // pack src [K][N] (fan_in x fan_out, plus an optional bias row at k = K_src)
    // rows of rank r into a K-major core-matrix image at base
    auto put = [&](size_t base, const double* src, uint32_t Ksrc, const double* bias, uint32_t K, uint32_t N,
                   uint32_t r, bool lo_part, size_t lo_base) {
      for (uint32_t kk = 0; kk < K; ++kk)
        for (uint32_t nl = 0; nl < NR; ++nl) {
          const uint32_t n = gcol(r, nl);
          double x = 0.0;
          if (kk < Ksrc) x = src[(size_t)kk * N + n];
          else if (kk == Ksrc && bias) x = bias[n];
          const size_t o = pack_offset(nl, kk, K, esz);
          if (bf && lo_part) {
            uint16_t hi, lo;
            f16_split(x, &hi, &lo);
            memcpy(&img[base + o], &hi, 2);
            memcpy(&img[lo_base + o], &lo, 2);
          } else if (bf) {
            uint16_t v = h16_rne(prec, (float)x);
            memcpy(&img[base + o], &v, 2);
          } else {
            uint32_t hi, lo;
            tf32_split(x, &hi, &lo);
            memcpy(&img[base + o], &hi, 4);
            if (lo_part) memcpy(&img[lo_base + o], &lo, 4);
          }
        }
    };
    for (uint32_t r = 0; r < ranks; ++r) {
      const size_t rb = (size_t)r * p.w_bytes;
      put(rb + p.off_b1, B1.data(), K0, nullptr, K0, H, r, lo1, rb + p.off_b1lo);
      for (uint32_t l = 1; l < NL; ++l) {
        const size_t base = rb + p.off_bh + (size_t)(l - 1) * p.stride_bh;
        put(base, m->W[e * L + l], H, bias_mma ? m->b[e * L + l] : nullptr, KH, H, r, loh, base + bh_bytes);
      }
    }
    // final layer: t = y_mean + y_scale (sum_j w_j relu(D_j + b_j) + b_out)
    //            = c' + sum_j w'_j max(D_j, -b_j),  w' = y_scale w,  c' = y_mean + y_scale (b_out + sum w b)
    // (b_j = 0 here when the bias is already in D: layer 1, or folded into the UMMA)
    const double* Wout = m->W[e * L + NL];
    const double bout = m->b[e * L + NL][0];
    const double* bl = (NL >= 2 && !bias_mma) ? m->b[e * L + NL - 1] : nullptr;
    double cacc = bout;
    std::vector<float> fw(H), fnb(H);
    for (uint32_t n = 0; n < H; ++n) {
      const double bj = bl ? bl[n] : 0.0;
      fnb[n] = (float)(-bj);
      // kernels with the bias in the UMMA evaluate w relu(x) as (w/2) x + (w/2) |x|
      fw[n] = (float)(m->y_scale * Wout[n] * (bias_mma ? 0.5 : 1.0));
      cacc += Wout[n] * bj;
      if (n < 128) { p.fin_nb[n] = fnb[n]; p.fin_w[n] = fw[n]; }  // parameter-bank copy (H <= 128 kernels)
    }
    p.c_out = (float)(m->y_mean + m->y_scale * cacc);
    for (uint32_t r = 0; r < ranks; ++r) {
      float* fwb = reinterpret_cast<float*>(&img[(size_t)r * p.w_bytes + p.off_fin]);
      for (uint32_t n = 0; n < H; ++n) { fwb[n] = fw[n]; fwb[H + n] = fnb[n]; }
    }
    if (!bias_mma)
      for (uint32_t l = 1; l + 1 < NL; ++l)
        for (uint32_t n = 0; n < H; ++n) p.hbias[l - 1][n] = (float)m->b[e * L + l][n];
    p.NL = NL;
    p.sbo_b1 = (K0 / (16 / esz)) * 128;
    p.sbo_bh = (KH / (16 / esz)) * 128;
    // a/b format: kind::f16 F16 = 0, BF16 = 1; kind::tf32 TF32 = 2
    const int fmt = prec == PREC_BF16 ? 1 : (prec == PREC_FP16 || prec == PREC_FP32H) ? 0 : 2;
    p.idesc = ki.pair ? make_idesc(fmt, H / 2, 2 * TILE_M) : make_idesc(fmt, H, TILE_M);
    p.P = P;
    mps[e] = p;
    imgs[e].swap(img);
  }
  // all members' images back to back (each 128-byte aligned, same size)
  const size_t wstride = imgs[0].size();
  std::vector<uint8_t> img(wstride * E);
  for (uint32_t e = 0; e < E; ++e) memcpy(img.data() + e * wstride, imgs[e].data(), wstride);

  // into the ring's other slot (complete on return): sweeps queued earlier keep
  // reading the weights their launch captured; no device-wide synchronisation
  void* dw = nullptr;
  surr_status urc = ring_upload(h, h->wring, img.data(), img.size(), nullptr, true, &dw);
  if (urc) return urc;
  for (uint32_t e = 0; e < E; ++e) {
    mps[e].w_gmem = (const uint8_t*)dw + e * wstride;
    for (uint32_t j = 0; j < (uint32_t)K0; ++j) {  // predict prologue constants (parameter bank)
      mps[e].zinv[j] = j < P ? (float)(1.0 / scale[j]) : 0.0f;
      mps[e].zc[j] = j < P ? (float)(-shift[j] / scale[j]) : 0.0f;
    }
  }
  h->members.swap(mps);
  h->rb_B1.swap(rb_B1);
  h->rb_W.swap(rb_W);
  h->rb_b.swap(rb_b);
  h->mp = h->members[0];
  h->hshift = shift;
  h->hscale = scale;
  h->wimg.swap(img);
  h->prec = prec;
  h->H = H;
  h->NL = NL;
  h->P = P;
  h->loaded = true;
  h->space_valid = false;
  h->c_values.clear();
  h->c_radix.clear();
  return SURR_OK;
}

surr_status surrogate_sweep(surrogate_t* h, const surr_space* space, uint32_t k, uint64_t* idx_dev, float* t_dev,
                            uint32_t* count_host, void* stream) {
  if (h && (!idx_dev || !t_dev)) return fail(h, SURR_E_INVALID_ARG, "null output");
  return sweep_common(h, space, k, idx_dev, t_dev, nullptr, count_host, (cudaStream_t)stream, false);
}

surr_status surrogate_sweep_records(surrogate_t* h, const surr_space* space, uint32_t k, surr_record* recs_dev,
                                    void* stream) {
  if (h && !recs_dev) return fail(h, SURR_E_INVALID_ARG, "null output");
  return sweep_common(h, space, k, nullptr, nullptr, recs_dev, nullptr, (cudaStream_t)stream, false);
}

surr_status surrogate_sweep_host(surrogate_t* h, const surr_space* space, uint32_t k, uint64_t* idx_host,
                                 float* t_host, uint32_t* count_host, void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!idx_host || !t_host) return fail(h, SURR_E_INVALID_ARG, "null output");
  if (k == 0 || k > SURR_K_MAX) return fail(h, SURR_E_INVALID_ARG, "k = %u outside 1..%u", k, SURR_K_MAX);
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaSetDevice(h->dev));
  if (!h->d_idx) {
    if (cudaMalloc(&h->d_idx, SURR_K_MAX * 8) != cudaSuccess || cudaMalloc(&h->d_t, SURR_K_MAX * 4) != cudaSuccess)
      return fail(h, SURR_E_OOM, "cudaMalloc");
  }
  surr_status rc = sweep_common(h, space, k, h->d_idx, h->d_t, nullptr, count_host, st, true);
  if (rc) return rc;
  CU(cudaMemcpyAsync(idx_host, h->d_idx, (size_t)k * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(t_host, h->d_t, (size_t)k * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return SURR_OK;
}

surr_status surrogate_eval_range(surrogate_t* h, const surr_space* space, float* t_dev, void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!h->loaded) return fail(h, SURR_E_NOT_LOADED, "no model loaded");
  if (!t_dev) return fail(h, SURR_E_INVALID_ARG, "null output");
  CU(cudaSetDevice(h->dev));
  surr_status rc = prepare_space(h, space, false, (cudaStream_t)stream);
  if (rc) return rc;
  h->launches = 0;
  if (h->sp.end == h->sp.begin) return SURR_OK;
  uint32_t lists = 0;
  return run_k1(h, h->sp.begin, h->sp.end, 1, MODE_DENSE, t_dev, nullptr, (cudaStream_t)stream, &lists);
}

surr_status surrogate_sweep_operands(surrogate_t* h, const surr_space* space, uint64_t stride, uint32_t* ops_dev,
                                     void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!h->loaded) return fail(h, SURR_E_NOT_LOADED, "no model loaded");
  if (!ops_dev || stride == 0) return fail(h, SURR_E_INVALID_ARG, "null output or stride 0");
  if (!(is16(h->prec) || h->prec == PREC_FP32H) || (h->prec == PREC_FP32H && h->NL != 2))
    return fail(h, SURR_E_UNSUPPORTED, "operand dump: FP16 / BF16 kernels and the 3xFP16 FP32-path kernel only");
  CU(cudaSetDevice(h->dev));
  surr_status rc = prepare_space(h, space, false, (cudaStream_t)stream);
  if (rc) return rc;
  h->launches = 0;
  if (h->sp.end == h->sp.begin) return SURR_OK;
  h->a0_dump = ops_dev;
  h->a0_stride = stride;
  uint32_t lists = 0;
  rc = run_k1(h, h->sp.begin, h->sp.end, 1, MODE_A0, nullptr, nullptr, (cudaStream_t)stream, &lists);
  h->a0_dump = nullptr;
  return rc;
}

surr_status surrogate_predict(surrogate_t* h, const float* x_dev, uint64_t n, float* t_dev, void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!h->loaded) return fail(h, SURR_E_NOT_LOADED, "no model loaded");
  h->launches = 0;
  if (n == 0) return SURR_OK;
  if (!x_dev || !t_dev) return fail(h, SURR_E_INVALID_ARG, "null buffer");
  CU(cudaSetDevice(h->dev));
  uint32_t lists = 0;
  return run_k1(h, 0, n, 1, MODE_PREDICT, t_dev, x_dev, (cudaStream_t)stream, &lists);
}

surr_status surrogate_merge_topk(surrogate_t* h, const surr_record* recs_dev, uint32_t lists, uint32_t k_in,
                                 uint32_t k, uint64_t* idx_dev, float* t_dev, surr_record* recs_out_dev,
                                 void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (k == 0 || k > SURR_K_MAX || k_in == 0 || k_in > SURR_K_MAX)
    return fail(h, SURR_E_INVALID_ARG, "k / k_in outside 1..%u", SURR_K_MAX);
  if ((lists && !recs_dev) || (!idx_dev && !t_dev && !recs_out_dev)) return fail(h, SURR_E_INVALID_ARG, "null buffer");
  CU(cudaSetDevice(h->dev));
  h->launches = 0;
  return launch_merge(h, recs_dev, lists, k_in, k, idx_dev, t_dev, recs_out_dev, (cudaStream_t)stream);
}

surr_status surrogate_decode_range(surrogate_t* h, const surr_space* space, uint64_t first, uint64_t n,
                                   uint8_t* digits_dev, void* stream) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  if (!h->loaded) return fail(h, SURR_E_NOT_LOADED, "load a model first (the table format follows its precision)");
  if (n && !digits_dev) return fail(h, SURR_E_INVALID_ARG, "null output");
  CU(cudaSetDevice(h->dev));
  surr_status rc = prepare_space(h, space, false, (cudaStream_t)stream);
  if (rc) return rc;
  if (first > h->card || n > h->card - first) return fail(h, SURR_E_INVALID_ARG, "range outside |S|");
  for (uint32_t j = 0; j < h->P; ++j)
    if (h->c_radix[j] > 256)
      return fail(h, SURR_E_UNSUPPORTED, "radix[%u] = %u: uint8 digits hold radices up to 256", j, h->c_radix[j]);
  h->launches = 0;
  if (n == 0) return SURR_OK;
  DecodeParams dp{};
  const KParams& s = h->sp;
  memcpy(dp.R, s.R, sizeof dp.R);
  for (uint32_t j = 0; j < h->P; ++j) dp.radix[j] = h->c_radix[j];
  dp.P = h->P;
  dp.spg = h->spg;
  dp.first = first; dp.n = n; dp.out = digits_dev;
  const uint32_t threads = 256;
  const uint64_t blocks = std::min<uint64_t>((n + threads - 1) / threads, 512);
  stride_digits(dp.R, blocks * threads, dp.dD);
  decode_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(dp);
  CU(cudaGetLastError());
  ++h->launches;
  return SURR_OK;
}

surr_status surrogate_debug_trace(surrogate_t* h, unsigned long long* trace_dev, uint32_t n) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  h->trace = trace_dev;
  h->trace_n = trace_dev ? n : 0;
  return SURR_OK;
}

surr_status surrogate_reset_cache(surrogate_t* h) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  h->space_valid = false;
  return SURR_OK;
}

surr_status surrogate_kernel_timing(surrogate_t* h, int enable) {
  if (!h) return fail(nullptr, SURR_E_INVALID_ARG, "null handle");
  h->timing = enable != 0;
  h->ev_used = 0;
  return SURR_OK;
}

surr_status surrogate_kernel_timing_get(surrogate_t* h, double* total_ms, uint32_t* launches) {
  if (!h || !total_ms || !launches) return fail(h, SURR_E_INVALID_ARG, "null argument");
  double tot = 0.0;
  for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
    CU(cudaEventSynchronize(h->ev[i + 1]));
    float ms = 0.0f;
    CU(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
    tot += ms;
  }
  *total_ms = tot;
  *launches = (uint32_t)(h->ev_used / 2);
  return SURR_OK;
}

surr_status surrogate_selftest_umma(int cuda_device, int precision, uint32_t n, uint32_t k, const float* a_host,
                                    const float* b_host, float* d_host) {
  surrogate* h = nullptr;
  if (!a_host || !b_host || !d_host) return fail(h, SURR_E_INVALID_ARG, "null argument");
  const bool bf = precision == SURR_PREC_BF16;
  if (!bf && precision != SURR_PREC_TF32) return fail(h, SURR_E_INVALID_ARG, "precision must be BF16 or TF32");
  const uint32_t kstep = bf ? 16 : 8;
  if (n < 32 || n > 256 || n % 32 || k == 0 || k % kstep || k > 256)
    return fail(h, SURR_E_UNSUPPORTED, "selftest shape N=%u K=%u", n, k);
  surr_status rc = check_device(h, cuda_device);
  if (rc) return rc;
  CU(cudaSetDevice(cuda_device));
  const uint32_t esz = bf ? 2 : 4;
  std::vector<uint8_t> img((size_t)n * k * esz, 0);
  for (uint32_t kk = 0; kk < k; ++kk)
    for (uint32_t j = 0; j < n; ++j) {
      const float x = b_host[(size_t)kk * n + j];
      const size_t o = pack_offset(j, kk, k, esz);
      if (bf) { uint16_t v = bf16_rne(x); memcpy(&img[o], &v, 2); }
      else { uint32_t v = tf32_rn(x); memcpy(&img[o], &v, 4); }
    }
  std::vector<uint32_t> a((size_t)128 * k, 0);  // TMEM image per row: bf16 pairs or tf32 words
  for (uint32_t r = 0; r < 128; ++r)
    for (uint32_t kk = 0; kk < k; ++kk) {
      const float x = a_host[(size_t)r * k + kk];
      if (bf) a[(size_t)r * k + kk / 2] |= (uint32_t)bf16_rne(x) << ((kk & 1) * 16);
      else a[(size_t)r * k + kk] = tf32_rn(x);
    }
  void *dA = nullptr, *dB = nullptr, *dD = nullptr;
  CU(cudaMalloc(&dA, a.size() * 4));
  CU(cudaMalloc(&dB, img.size()));
  CU(cudaMalloc(&dD, (size_t)128 * n * 4));
  CU(cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dB, img.data(), img.size(), cudaMemcpyHostToDevice));
  const uint32_t acols = bf ? k / 2 : k;
  const uint32_t idesc = make_idesc(bf ? 1 : 2, n, TILE_M);
  const uint32_t sbo = (k / (16 / esz)) * 128;
  const size_t smem = align_up(img.size(), 128) + 64;
  CU(cudaFuncSetAttribute((const void*)umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  umma_selftest_kernel<<<1, 128, smem>>>((const uint32_t*)dA, k, acols, (const uint8_t*)dB, (uint32_t)img.size(),
                                          (float*)dD, n, bf ? 1 : 0, idesc, sbo);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(d_host, dD, (size_t)128 * n * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return SURR_OK;
}

surr_status surrogate_train(surrogate_t* h, const uint32_t* widths, uint32_t E, double* const* W, double* const* b,
                            const double* X, const double* y, uint64_t n, const uint32_t* perms,
                            const surr_train_hyper* hy, double* loss_history, uint32_t* epochs_run,
                            uint32_t* stop_reason) {
  if (!h || !widths || !W || !b || !X || !y || !hy || !loss_history || !epochs_run || !stop_reason)
    return fail(h, SURR_E_INVALID_ARG, "null argument");
  if (E == 0) return fail(h, SURR_E_INVALID_ARG, "E == 0");
  for (uint32_t l = 0; l < 3 * E; ++l)
    if (!W[l] || !b[l]) return fail(h, SURR_E_INVALID_ARG, "null layer %u", l);
  const uint32_t F = widths[0], H = widths[1];
  if (widths[2] != H || widths[3] != 1)
    return fail(h, SURR_E_UNSUPPORTED, "training supports F-H-H-1 nets (two equal hidden layers)");
  if (F < 1 || F > (uint32_t)TR_FMAX) return fail(h, SURR_E_UNSUPPORTED, "F = %u outside 1..%d", F, TR_FMAX);
  if (H != 32 && H != 64 && H != 128) return fail(h, SURR_E_UNSUPPORTED, "H = %u not in {32, 64, 128}", H);
  const uint32_t C = H / TR_CPC;
  if (n == 0 || n > 0xFFFFFFFFull) return fail(h, SURR_E_INVALID_ARG, "n = %llu", (unsigned long long)n);
  if (hy->batch_size < 1 || hy->batch_size > (uint32_t)TR_BMAX || hy->max_epochs < 1 || !(hy->lr0 > 0.0) ||
      !(hy->beta1 >= 0.0 && hy->beta1 < 1.0) || !(hy->beta2 >= 0.0 && hy->beta2 < 1.0) || !(hy->eps > 0.0) ||
      !(hy->alpha >= 0.0))
    return fail(h, SURR_E_INVALID_ARG, "hyperparameters outside their domain");
  const uint64_t nperm = (uint64_t)E * hy->max_epochs * n;
  if (perms)
    for (uint64_t i = 0; i < nperm; ++i)
      if (perms[i] >= n) return fail(h, SURR_E_INVALID_ARG, "perms[%llu] = %u >= n", (unsigned long long)i, perms[i]);
  CU(cudaSetDevice(h->dev));
  // member image: W1 [F][H], b1, W2 [H][H], b2, W3 [H], b3, padded to 4 floats
  const size_t sizes[6] = {(size_t)F * H, H, (size_t)H * H, H, H, 1};
  size_t off[7] = {0};
  for (int i = 0; i < 6; ++i) off[i + 1] = off[i] + sizes[i];
  const size_t pstride = align_up(off[6], 4);
  std::vector<float> hp(pstride * E, 0.0f), hx((size_t)n * F), hyv(n);
  for (uint32_t e = 0; e < E; ++e)
    for (int i = 0; i < 6; ++i) {
      const double* src = (i % 2 == 0) ? W[3 * e + i / 2] : b[3 * e + i / 2];
      for (size_t j = 0; j < sizes[i]; ++j) hp[e * pstride + off[i] + j] = (float)src[j];
    }
  for (size_t i = 0; i < (size_t)n * F; ++i) hx[i] = (float)X[i];
  for (uint64_t i = 0; i < n; ++i) hyv[i] = (float)y[i];
  float *dp = nullptr, *dx = nullptr, *dy = nullptr, *dmv = nullptr;
  uint32_t *dperm = nullptr, *dres = nullptr;
  double* dloss = nullptr;
  const size_t perm_bytes = perms ? nperm * 4 : 0;
  auto release = [&]() {
    cudaFree(dp); cudaFree(dx); cudaFree(dy); cudaFree(dmv); cudaFree(dperm); cudaFree(dres); cudaFree(dloss);
  };
  if (cudaMalloc(&dp, hp.size() * 4) != cudaSuccess || cudaMalloc(&dx, hx.size() * 4) != cudaSuccess ||
      cudaMalloc(&dy, hyv.size() * 4) != cudaSuccess ||
      cudaMalloc(&dmv, (size_t)E * C * 2 * H * TR_CPC * 4) != cudaSuccess ||
      cudaMalloc(&dres, (size_t)E * 12) != cudaSuccess ||
      cudaMalloc(&dloss, (size_t)E * hy->max_epochs * 8) != cudaSuccess ||
      (perms && cudaMalloc(&dperm, perm_bytes) != cudaSuccess)) {
    release();
    return fail(h, SURR_E_OOM, "cudaMalloc (training buffers)");
  }
  surr_status rc = SURR_OK;
  do {
#define TCU(call)                                                                          \
  {                                                                                        \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) { rc = fail(h, SURR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); break; } \
  }
    TCU(cudaMemcpy(dp, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice));
    TCU(cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
    TCU(cudaMemcpy(dy, hyv.data(), hyv.size() * 4, cudaMemcpyHostToDevice));
    if (perms) TCU(cudaMemcpy(dperm, perms, perm_bytes, cudaMemcpyHostToDevice));
    TrainParams tp{};
    tp.X = dx; tp.y = dy; tp.perms = dperm;
    tp.n = (uint32_t)n; tp.F = F; tp.B = hy->batch_size; tp.E = E;
    tp.max_epochs = hy->max_epochs; tp.n_iter_no_change = hy->n_iter_no_change;
    tp.alpha = (float)hy->alpha; tp.beta1 = (float)hy->beta1; tp.beta2 = (float)hy->beta2;
    tp.lr0 = (float)hy->lr0; tp.eps = (float)hy->eps; tp.tol = hy->tol;
    tp.params = dp;
    tp.pstride = (uint32_t)pstride;
    tp.oW1 = (uint32_t)off[0]; tp.ob1 = (uint32_t)off[1]; tp.oW2 = (uint32_t)off[2];
    tp.ob2 = (uint32_t)off[3]; tp.oW3 = (uint32_t)off[4]; tp.ob3 = (uint32_t)off[5];
    tp.mv = dmv; tp.loss_hist = dloss; tp.result = dres;
    unsigned long long* dprof = nullptr;  // development: SURR_TRAIN_PROF=1 prints per-phase cycles
    if (getenv("SURR_TRAIN_PROF") && cudaMalloc(&dprof, 16 * 8) == cudaSuccess) {
      cudaMemset(dprof, 0, 16 * 8);
      tp.prof = dprof;
    }
    const bool push = E > 1;  // DSMEM push exchange for ensembles, pull for one member (measured)
    const void* fn = H == 32  ? (push ? (const void*)&train_kernel<32, true> : (const void*)&train_kernel<32, false>)
                     : H == 64 ? (push ? (const void*)&train_kernel<64, true> : (const void*)&train_kernel<64, false>)
                               : (push ? (const void*)&train_kernel<128, true> : (const void*)&train_kernel<128, false>);
    const size_t smem = H == 32 ? sizeof(TrainSmem<32>) : H == 64 ? sizeof(TrainSmem<64>) : sizeof(TrainSmem<128>);
    if (smem > SMEM_MAX) { rc = fail(h, SURR_E_UNSUPPORTED, "training shared memory %zu B", smem); break; }
    TCU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C * E, 1, 1);
    cfg.blockDim = dim3(TR_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = nullptr;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&tp};
    TCU(cudaLaunchKernelExC(&cfg, fn, args));
    h->launches = 1;
    TCU(cudaDeviceSynchronize());
    if (dprof) {
      unsigned long long pr[16];
      cudaMemcpy(pr, dprof, sizeof pr, cudaMemcpyDeviceToHost);
      cudaFree(dprof);
      fprintf(stderr, "train phases (cycles, CTA 0):");
      for (int i = 0; i < 14; ++i) fprintf(stderr, " %d:%llu", i, pr[i]);
      fprintf(stderr, "\n");
    }
    std::vector<uint32_t> res((size_t)E * 3);
    TCU(cudaMemcpy(res.data(), dres, res.size() * 4, cudaMemcpyDeviceToHost));
    TCU(cudaMemcpy(hp.data(), dp, hp.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<double> lh((size_t)E * hy->max_epochs);
    TCU(cudaMemcpy(lh.data(), dloss, lh.size() * 8, cudaMemcpyDeviceToHost));
    for (uint32_t e = 0; e < E && rc == SURR_OK; ++e)
      for (uint32_t p = 0; p < res[3 * e]; ++p)
        if (!std::isfinite(lh[(size_t)e * hy->max_epochs + p])) {
          // a diverged fit (S: training aborts on a non-finite loss): no weights are returned
          rc = fail(h, SURR_E_RANGE, "member %u: non-finite training loss in epoch %u (divergence)", e, p + 1);
          break;
        }
    if (rc != SURR_OK) break;
    for (uint32_t e = 0; e < E; ++e) {
      for (uint32_t p = 0; p < res[3 * e]; ++p)
        loss_history[(size_t)e * hy->max_epochs + p] = lh[(size_t)e * hy->max_epochs + p];
      for (int i = 0; i < 6; ++i) {
        double* dst = (i % 2 == 0) ? W[3 * e + i / 2] : b[3 * e + i / 2];
        for (size_t j = 0; j < sizes[i]; ++j) dst[j] = (double)hp[e * pstride + off[i] + j];
      }
      epochs_run[e] = res[3 * e];
      stop_reason[e] = res[3 * e + 1];
    }
#undef TCU
  } while (0);
  release();
  return rc;
}

}  // extern "C"
