/*
 * ORACLE — test infrastructure only (tests/, smoke(), bench.py cpu_baseline).
 *
 * Plain-C restatement of the reference's seeded shuffle so large-n parity
 * (n = 1e6, pinned by a SHA-256 computed from the reference) runs in
 * milliseconds instead of the reference's ~1.5 s pure-Python loop.
 *   splitmix64           reference packed_data.py:226-238
 *   oracle_permutation   reference packed_data.py:257-282
 * Rejection threshold floor(2^64/b)*b is formed with unsigned __int128 here
 * (independent of the product's modular-arithmetic formulation).
 * Also: oracle_gather, a scalar loop restating get_sample (:196-203) for the
 * cpu_baseline leg of bench.py.
 */
#include <stdint.h>
#include <string.h>

static uint64_t mix(uint64_t *st) {
  *st += 0x9E3779B97F4A7C15ull;
  uint64_t z = *st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_permutation(uint64_t n, uint64_t seed, uint64_t *order) {
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  uint64_t st = seed;
  for (uint64_t i = n; i-- > 1;) {
    unsigned __int128 b = (unsigned __int128)(i + 1);
    unsigned __int128 lim = (((unsigned __int128)1 << 64) / b) * b;
    uint64_t x;
    do {
      x = mix(&st);
    } while ((unsigned __int128)x >= lim);
    uint64_t j = x % (i + 1);
    uint64_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
}

/* inputs/targets [B, L] int64 from a width-byte little-endian payload. Returns -1 on a bad id. */
int oracle_gather(const uint8_t *payload, int width, uint64_t token_count, const uint64_t *ids,
                  int B, int64_t L, int64_t *inputs, int64_t *targets) {
  uint64_t nsamp = token_count ? (token_count - 1) / (uint64_t)L : 0;
  for (int b = 0; b < B; ++b) {
    if (ids[b] >= nsamp) return -1;
    uint64_t base = ids[b] * (uint64_t)L;
    for (int64_t t = 0; t <= L; ++t) {
      uint64_t v = 0;
      memcpy(&v, payload + (base + (uint64_t)t) * (uint64_t)width, (size_t)width);
      if (t < L) inputs[(int64_t)b * L + t] = (int64_t)v;
      if (t > 0) targets[(int64_t)b * L + t - 1] = (int64_t)v;
    }
  }
  return 0;
}
