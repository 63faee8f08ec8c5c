/* Plain C use of the C ABI (include/surrogate.h): no Python, no torch.
 * Loads a 14-32-32-1 net given as plain arrays (seeded values generated here),
 * sweeps the 2^14-config tiny space (gang {100, 1000} x vector {32, 384} per
 * kernel, PAPER.md:253-266 endpoints) for the 3 fastest predicted configs with
 * host outputs, and prints them.  Exit status: 0 ok, 2 no sm_100 device,
 * 1 any other error.
 *
 *   gcc -O2 -I include examples/c_api_example.c -L paper_2306_14011_b200 -lsurrogate \
 *       -Wl,-rpath,$PWD/paper_2306_14011_b200 -o /tmp/c_api_example && /tmp/c_api_example
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "surrogate.h"

static uint64_t state = 0x2306014011ull;
static double urand(void) { /* SplitMix64 -> [0, 1) */
  uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
  enum { P = 14, H = 32, L = 3 };
  uint32_t radix[P];
  double values[2 * P];
  for (int j = 0; j < P; ++j) {
    radix[j] = 2;
    values[2 * j] = (j % 2 == 0) ? 100.0 : 32.0;  /* gang / vector endpoints */
    values[2 * j + 1] = (j % 2 == 0) ? 1000.0 : 384.0;
  }
  const uint32_t widths[L + 1] = {P, H, H, 1};
  static double W0[P * H], W1[H * H], W2[H], b0[H], b1[H], b2[1];
  double* Wl[L] = {W0, W1, W2};
  double* bl[L] = {b0, b1, b2};
  for (int l = 0; l < L; ++l) {
    const double bound = l == 0 ? 0.38 : l == 1 ? 0.3 : 0.42; /* ~ Glorot sqrt(6 / (fan_in + fan_out)) */
    for (uint32_t i = 0; i < widths[l] * widths[l + 1]; ++i) Wl[l][i] = (2.0 * urand() - 1.0) * bound;
    for (uint32_t i = 0; i < widths[l + 1]; ++i) bl[l][i] = (2.0 * urand() - 1.0) * bound;
  }
  double shift[P], scale[P];
  for (int j = 0; j < P; ++j) { /* z in [-1, 1] over each list */
    shift[j] = 0.5 * (values[2 * j] + values[2 * j + 1]);
    scale[j] = 0.5 * (values[2 * j + 1] - values[2 * j]);
  }
  const double* const Wc[L] = {W0, W1, W2};
  const double* const bc[L] = {b0, b1, b2};
  surr_model m = {L, widths, Wc, bc, shift, scale, 1.4, 0.3, 0, NULL, 1, SURR_PREC_FP32};
  surr_space sp = {P, radix, values, 0, 0};

  uint64_t n = 0;
  if (surrogate_space_size(&sp, &n) != SURR_OK) return 1;
  surrogate_t* h = NULL;
  surr_status rc = surrogate_create(0, &h);
  if (rc == SURR_E_NO_DEVICE) {
    printf("no sm_100 device: %s\n", surrogate_last_error(h));
    surrogate_destroy(h);
    return 2;
  }
  if (rc != SURR_OK || surrogate_load_weights(h, &m) != SURR_OK) {
    printf("error: %s\n", surrogate_last_error(h));
    surrogate_destroy(h);
    return 1;
  }
  uint64_t idx[3];
  float t[3];
  uint32_t cnt = 0;
  if (surrogate_sweep_host(h, &sp, 3, idx, t, &cnt, NULL) != SURR_OK) {
    printf("error: %s\n", surrogate_last_error(h));
    surrogate_destroy(h);
    return 1;
  }
  printf("space %llu configs, top %u:\n", (unsigned long long)n, cnt);
  for (uint32_t r = 0; r < cnt; ++r) printf("%llu %.9g\n", (unsigned long long)idx[r], (double)t[r]);
  surrogate_destroy(h);
  return 0;
}
