/* Fast path of synth/gen.py weight_values(): the same counter hash, OpenMP over elements.
 * Input generator only (no method arithmetic).  Built by synth/build_gen.py. */
#include <math.h>
#include <stdint.h>

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void synth_weight_values(float* out, uint64_t tid, uint64_t start, uint64_t count, uint64_t seed, int exp2) {
  const uint64_t base = (tid << 40) + (seed + 1ull) * 0x9E3779B97F4A7C15ull;
  const float scale = ldexpf(1.0f, exp2);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)count; ++i) {
    const uint64_t u = mix64(base + start + (uint64_t)i);
    out[i] = (float)(2 * (int)(u >> 56) - 255) * scale;
  }
}
