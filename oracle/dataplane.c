/* ORACLE — test infrastructure only.  Never linked into, imported by, or
 * called from the product path (paper_2502_09922_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg load it, as the
 * checker.
 *
 * CPU restatement of the λPipe data plane:
 *   lp_ref_fill      the synthetic bf16 generator (lp_image.cu gen_bf16)
 *   lp_ref_checksum  the per-block checksum     (lp_image.cu checksum_kernel)
 *   lp_ref_execute   executes a schedule as the reference defines it: steps in
 *                    order (multicast.py:91-124 arrival semantics), every
 *                    transfer (step,sender,receiver,block) of
 *                    schedule_to_lines (multicast.py:546-551) copies the
 *                    block's bytes sender->receiver; a sender must hold the
 *                    block at the start of the step (causality, the check of
 *                    multicast.py:507-509).  Transfers of one step run in
 *                    parallel on `threads` OpenMP threads, one barrier per
 *                    step (the lockstep model of simengine.py:594-596).
 * Parity pin: the schedules it executes are the reference's own lines
 * (tests/golden/, dumped by tests/golden/make_golden.py from the reference).
 * Byte content has no reference (the paper's RDMC data plane is not vendored,
 * SURVEY.md §8c): delivered-bytes parity = receiver block == source block.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  uint32_t bias = ((u >> 16) & 1u) + 0x7FFFu;
  return (uint16_t)((u + bias) >> 16);
}

void lp_ref_fill(uint16_t* out, int64_t numel, int tensor_id, uint64_t seed, int kind, int scale_exp) {
  if (kind == 1) { for (int64_t i = 0; i < numel; ++i) out[i] = 0x3F80; return; }
  if (kind == 2) { memset(out, 0, (size_t)numel * 2); return; }
  const float scale = ldexpf(1.0f, scale_exp - 15);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < numel; ++i) {
    uint64_t z = mix64(seed + ((uint64_t)(tensor_id + 1) << 40) + (uint64_t)i);
    int v = (int)(z >> 48) - 32768;
    out[i] = f32_to_bf16_rne((float)v * scale);
  }
}

uint64_t lp_ref_checksum(const uint8_t* base, int64_t len) {
  const int64_t nw = len / 8;
  uint64_t acc = 0;
  #pragma omp parallel for reduction(+:acc) schedule(static)
  for (int64_t k = 0; k < nw; ++k) {
    uint64_t w;
    memcpy(&w, base + 8 * k, 8);
    acc += mix64(w ^ ((uint64_t)k * 0x9E3779B97F4A7C15ull));
  }
  return acc;
}

/* xfers: n x 4 (step, sender, receiver, block), sorted by step.
 * holds: n_nodes x n_blocks bytes, 1 where the node holds the block at start.
 * returns 0, or -(1 + index) of the first causality violation. */
int64_t lp_ref_execute(int n_nodes, uint8_t** images, int n_blocks, const int64_t* off,
                       const int64_t* len, const int32_t* xfers, int64_t n, uint8_t* holds,
                       int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  int64_t i = 0;
  while (i < n) {
    int64_t j = i;
    while (j < n && xfers[4 * j] == xfers[4 * i]) ++j;
    for (int64_t t = i; t < j; ++t) {
      const int32_t* x = xfers + 4 * t;
      if (x[1] < 0 || x[1] >= n_nodes || x[2] < 0 || x[2] >= n_nodes || x[3] < 0 || x[3] >= n_blocks)
        return -(1 + t);
      if (!holds[(int64_t)x[1] * n_blocks + x[3]]) return -(1 + t);
    }
    /* one step: chunk every transfer so all threads help on big blocks */
    const int64_t CH = 8 << 20;
    int64_t total_chunks = 0;
    for (int64_t t = i; t < j; ++t) total_chunks += (len[xfers[4 * t + 3]] + CH - 1) / CH;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < total_chunks; ++c) {
      int64_t rem = c, t = i;
      for (; t < j; ++t) {
        int64_t nc = (len[xfers[4 * t + 3]] + CH - 1) / CH;
        if (rem < nc) break;
        rem -= nc;
      }
      const int32_t* x = xfers + 4 * t;
      int64_t lo = rem * CH, bl = len[x[3]];
      int64_t cnt = bl - lo < CH ? bl - lo : CH;
      memcpy(images[x[2]] + off[x[3]] + lo, images[x[1]] + off[x[3]] + lo, (size_t)cnt);
    }
    for (int64_t t = i; t < j; ++t) holds[(int64_t)xfers[4 * t + 2] * n_blocks + xfers[4 * t + 3]] = 1;
    i = j;
  }
  return 0;
}
