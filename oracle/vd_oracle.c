/* CPU ORACLE — test infrastructure only (see vd_oracle.h). Never part of the
 * product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load this library, and only as the checker.
 *
 * Every function restates the reference algorithm with `double` path
 * metrics exactly as the reference computes them (same operations, same
 * order), so results are bit-identical to the reference for ANY real-valued
 * input, and in particular for integer-valued (int8) inputs. File:line
 * citations are into /root/reference/proj.
 *
 * Parity pinned by tests/test_oracle.py (reference KATs + golden fixtures
 * produced by the reference itself, tests/golden/make_golden.py).
 */
#include "vd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

const char* vdo_last_error(void) { return g_err; }

/* splitmix64 finalizer — src/channel.cpp:85-90. */
uint64_t vdo_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* src/channel.cpp:16-20. */
double vdo_sigma_from_ebn0(double ebn0_db, double rate) {
  const double ebn0 = pow(10.0, ebn0_db / 10.0);
  return sqrt(1.0 / (2.0 * rate * ebn0));
}

/* ---- trellis: src/trellis.cpp:38-101 ------------------------------------ */

static int popcount32(uint32_t x) { return __builtin_popcount(x); }

static int validate_spec(int k, int b, const uint32_t* polys) {
  /* src/trellis.cpp:38-53 */
  if (k < 2) return fail("constraint length must be >= 2");
  if (b < 2) return fail("need at least 2 outputs per bit");
  if (k > 16) return fail("constraint length too large");
  const uint32_t mask = (1u << k) - 1;
  for (int i = 0; i < b; ++i) {
    if (polys[i] == 0) return fail("zero generator polynomial");
    if ((polys[i] & ~mask) != 0) return fail("generator polynomial wider than K bits");
  }
  return 0;
}

int vdo_trellis(int k, int b, const uint32_t* polys, uint32_t* next, uint32_t* out, uint32_t* pred,
                uint32_t* in_out, int* complement_paired) {
  if (validate_spec(k, b, polys)) return 1;
  const uint32_t s = 1u << (k - 1);
  /* next/out: src/trellis.cpp:65-79. Register = input bit on top of state. */
  for (uint32_t st = 0; st < s; ++st) {
    for (uint32_t u = 0; u < 2; ++u) {
      const uint32_t reg = (u << (k - 1)) | st;
      uint32_t bo = 0;
      for (int i = 0; i < b; ++i) bo |= (uint32_t)(popcount32(polys[i] & reg) & 1) << (b - 1 - i);
      next[st * 2 + u] = (u << (k - 2)) | (st >> 1);
      out[st * 2 + u] = bo;
    }
  }
  /* pred/in_out: src/trellis.cpp:81-91 (low = 0 when S == 2). */
  const uint32_t low_mask = s / 2 - 1;
  for (uint32_t j = 0; j < s; ++j) {
    const uint32_t low = (s == 2) ? 0 : (j & low_mask);
    const uint32_t u = j >> (k - 2); /* branch_input, trellis.hpp:57-59 */
    for (uint32_t w = 0; w < 2; ++w) {
      const uint32_t i = low * 2 + w;
      pred[j * 2 + w] = i;
      in_out[j * 2 + w] = out[i * 2 + u];
    }
  }
  /* src/trellis.cpp:93-100 */
  const uint32_t ones = (1u << b) - 1;
  int cp = 1;
  for (uint32_t st = 0; st < s; ++st) {
    if ((out[st * 2] ^ out[st * 2 + 1]) != ones) {
      cp = 0;
      break;
    }
  }
  *complement_paired = cp;
  return 0;
}

/* ---- decoder: src/decoder.cpp ------------------------------------------- */

typedef struct {
  int k, b, s;
  uint32_t* in_out;
} code_t;

static int code_init(code_t* c, int k, int b, const uint32_t* polys) {
  if (validate_spec(k, b, polys)) return 1;
  c->k = k;
  c->b = b;
  c->s = 1 << (k - 1);
  const size_t n2 = (size_t)c->s * 2;
  uint32_t* next = malloc(sizeof(uint32_t) * n2);
  uint32_t* out = malloc(sizeof(uint32_t) * n2);
  uint32_t* pred = malloc(sizeof(uint32_t) * n2);
  c->in_out = malloc(sizeof(uint32_t) * n2);
  int cp;
  vdo_trellis(k, b, polys, next, out, pred, c->in_out, &cp);
  free(next);
  free(out);
  free(pred);
  return 0;
}

static void code_free(code_t* c) { free(c->in_out); }

/* branch_metric (:22-30) + fill_stage_table (:41-51): first 2^(B-1) entries
 * direct, the rest by complement symmetry. */
static void fill_stage_table(const double* llr_t, int b, double* table) {
  const uint32_t half = 1u << (b - 1);
  const uint32_t mask = (1u << b) - 1;
  for (uint32_t bo = 0; bo < half; ++bo) {
    double m = 0.0;
    for (int i = 0; i < b; ++i) {
      const int bit = (bo >> (b - 1 - i)) & 1;
      m += bit ? -llr_t[i] : llr_t[i];
    }
    table[bo] = m;
  }
  for (uint32_t bo = half; bo <= mask; ++bo) table[bo] = -table[bo ^ mask];
}

/* acs_stage (:53-76): strict '>' so exact ties take the second predecessor. */
static void acs_stage(const code_t* c, const double* sp, const double* table, double* sc, uint16_t* pi_col) {
  const uint32_t low_mask = (uint32_t)(c->s / 2 - 1);
  for (int j = 0; j < c->s; ++j) {
    const uint32_t i1 = ((uint32_t)j & low_mask) << 1;
    const uint32_t i2 = i1 | 1;
    const double s1 = sp[i1] + table[c->in_out[2 * j]];
    const double s2 = sp[i2] + table[c->in_out[2 * j + 1]];
    if (s1 > s2) {
      sc[j] = s1;
      pi_col[j] = (uint16_t)i1;
    } else {
      sc[j] = s2;
      pi_col[j] = (uint16_t)i2;
    }
  }
}

/* argmax_state (:80-90): first strict max, i.e. lowest index on ties. */
static int argmax_state(const double* sigma, int s) {
  int best = 0;
  double best_v = sigma[0];
  for (int j = 1; j < s; ++j) {
    if (sigma[j] > best_v) {
      best_v = sigma[j];
      best = j;
    }
  }
  return best;
}

typedef struct {
  int f, v1, v2, f0, start;
  uint64_t seed;
} frame_cfg_t;

static int validate_cfg(const frame_cfg_t* cfg) {
  /* FrameConfig::validate, :10-20 (period 1 as framed_decode calls it, :244) */
  if (cfg->f < 1) return fail("frame size f must be >= 1");
  if (cfg->v1 < 0 || cfg->v2 < 0) return fail("overlaps must be >= 0");
  if (cfg->f0 < 0 || cfg->f0 > cfg->f) return fail("f0 must be in [0, f]");
  return 0;
}

/* llr accessor: either double or int8 storage, stage-major t*B+b. */
typedef struct {
  const double* d;
  const int8_t* q;
} llr_src_t;

static void load_stage(const llr_src_t* src, int b, int64_t t, double* out) {
  for (int i = 0; i < b; ++i) out[i] = src->d ? src->d[t * b + i] : (double)src->q[t * b + i];
}

/* decode_frame, :170-237. */
static void decode_frame(const code_t* c, const llr_src_t* src, int64_t n, const frame_cfg_t* cfg, int64_t frame,
                         uint8_t* out_bits, double* sigma_out) {
  const int s = c->s;
  const int64_t out_lo = frame * cfg->f;
  const int64_t out_hi = out_lo + cfg->f < n ? out_lo + cfg->f : n;
  const int64_t beg = out_lo - cfg->v1 > 0 ? out_lo - cfg->v1 : 0;
  const int64_t end = out_hi + cfg->v2 < n ? out_hi + cfg->v2 : n;
  const int64_t len = end - beg;

  /* subframes, :182-191 */
  const int64_t step = cfg->f0 > 0 ? cfg->f0 : (out_hi - out_lo);
  const int64_t num_sub = (out_hi - out_lo + step - 1) / step;
  int64_t* start_stage = malloc(sizeof(int64_t) * (size_t)num_sub);
  uint16_t* start_state = calloc((size_t)num_sub, sizeof(uint16_t));
  for (int64_t sb = 0; sb < num_sub; ++sb) {
    const int64_t sub_hi = out_lo + (sb + 1) * step < out_hi ? out_lo + (sb + 1) * step : out_hi;
    const int64_t e = sub_hi + cfg->v2 < end ? sub_hi + cfg->v2 : end;
    start_stage[sb] = e - 1 - beg;
  }

  uint16_t* pi = malloc(sizeof(uint16_t) * (size_t)s * (size_t)len);
  double* sp = calloc((size_t)s, sizeof(double)); /* sigma_0 = 0, :195 */
  double* sc = malloc(sizeof(double) * (size_t)s);
  double table[256]; /* 2^B entries; B <= 8 enforced by callers of the oracle */
  double llr_t[16];

  /* forward pass + argmax at start stages, :199-212 */
  int64_t next_record = 0;
  for (int64_t t = 0; t < len; ++t) {
    load_stage(src, c->b, beg + t, llr_t);
    fill_stage_table(llr_t, c->b, table);
    acs_stage(c, sp, table, sc, pi + (size_t)t * s);
    double* tmp = sp;
    sp = sc;
    sc = tmp;
    while (next_record < num_sub && start_stage[next_record] == t) {
      start_state[next_record] = (uint16_t)argmax_state(sp, s);
      ++next_record;
    }
  }
  if (sigma_out) memcpy(sigma_out, sp, sizeof(double) * (size_t)s);

  /* traceback per subframe, :214-236 */
  for (int64_t sb = 0; sb < num_sub; ++sb) {
    const int64_t sub_lo = out_lo + sb * step;
    const int64_t sub_hi = sub_lo + step < out_hi ? sub_lo + step : out_hi;
    int state;
    if (cfg->f0 > 0 && cfg->start == 1 && start_stage[sb] < len - 1) {
      state = (int)(vdo_mix_seed(cfg->seed, (uint64_t)frame * 0x10001ull + (uint64_t)sb) % (uint64_t)s);
    } else {
      state = start_state[sb];
    }
    for (int64_t t = start_stage[sb]; t >= sub_lo - beg; --t) {
      const int64_t stage = beg + t;
      if (stage < sub_hi) out_bits[stage] = (uint8_t)(state >> (c->k - 2));
      state = pi[(size_t)t * s + state];
    }
  }
  free(pi);
  free(sp);
  free(sc);
  free(start_stage);
  free(start_state);
}

static int framed_common(int k, int b, const uint32_t* polys, const llr_src_t* src, int64_t n, int f, int v1,
                         int v2, int f0, int start, uint64_t seed, int64_t fb, int64_t fe, uint8_t* bits_out,
                         int64_t* stats, double* sigma_out) {
  code_t c;
  if (code_init(&c, k, b, polys)) return 1;
  /* check_block, :92-97 */
  if (n < 1) {
    code_free(&c);
    return fail("empty llr block");
  }
  const frame_cfg_t cfg = {f, v1, v2, f0, start, seed};
  if (validate_cfg(&cfg)) {
    code_free(&c);
    return 1;
  }
  const int64_t num_frames = (n + f - 1) / f;
  if (fe < 0 || fe > num_frames) fe = num_frames;
  for (int64_t m = fb; m < fe; ++m) {
    decode_frame(&c, src, n, &cfg, m, bits_out, sigma_out ? sigma_out + (size_t)m * c.s : NULL);
  }
  if (stats) {
    /* :256-265 */
    stats[0] = num_frames;
    stats[1] = 0;
    stats[2] = 0;
    for (int64_t m = 0; m < num_frames; ++m) {
      const int64_t out_lo = m * f;
      const int64_t out_hi = out_lo + f < n ? out_lo + f : n;
      const int64_t beg = out_lo - v1 > 0 ? out_lo - v1 : 0;
      const int64_t end = out_hi + v2 < n ? out_hi + v2 : n;
      stats[1] += end - beg;
      const int64_t step = f0 > 0 ? f0 : (out_hi - out_lo);
      stats[2] += (out_hi - out_lo + step - 1) / step;
    }
  }
  code_free(&c);
  return 0;
}

int vdo_framed_decode_f64(int k, int b, const uint32_t* polys, const double* llr, int64_t n, int f, int v1, int v2,
                          int f0, int start, uint64_t seed, uint8_t* bits_out, int64_t* stats, double* sigma_out) {
  const llr_src_t src = {llr, NULL};
  return framed_common(k, b, polys, &src, n, f, v1, v2, f0, start, seed, 0, -1, bits_out, stats, sigma_out);
}

int vdo_framed_decode_i8(int k, int b, const uint32_t* polys, const int8_t* llr, int64_t n, int f, int v1, int v2,
                         int f0, int start, uint64_t seed, uint8_t* bits_out, int64_t* stats, double* sigma_out) {
  const llr_src_t src = {NULL, llr};
  return framed_common(k, b, polys, &src, n, f, v1, v2, f0, start, seed, 0, -1, bits_out, stats, sigma_out);
}

int vdo_framed_decode_range_i8(int k, int b, const uint32_t* polys, const int8_t* llr, int64_t n, int f, int v1,
                               int v2, int f0, int start, uint64_t seed, int64_t frame_begin, int64_t frame_end,
                               uint8_t* bits_out) {
  const llr_src_t src = {NULL, llr};
  return framed_common(k, b, polys, &src, n, f, v1, v2, f0, start, seed, frame_begin, frame_end, bits_out, NULL,
                       NULL);
}

/* serial_decode, :101-129 — identical to one frame with f >= n, v1 = v2 = 0. */
int vdo_serial_decode_f64(int k, int b, const uint32_t* polys, const double* llr, int64_t n, uint8_t* bits_out,
                          double* sigma_out) {
  if (n < 1) return fail("empty llr block");
  if (n > 0x7fffffff) return fail("block too long for the oracle");
  const llr_src_t src = {llr, NULL};
  return framed_common(k, b, polys, &src, n, (int)n, 0, 0, 0, 0, 0, 0, -1, bits_out, NULL, sigma_out);
}

/* ---- channel / codec: src/channel.cpp, src/codec.cpp --------------------- */

/* std::mt19937_64 (the standard MT19937-64 parameters), restated. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64_t* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= A;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* random_bits, channel.cpp:68-83: LSB-first bits of successive 64-bit draws. */
void vdo_random_bits(int64_t n, uint64_t seed, uint8_t* bits) {
  mt64_t* g = malloc(sizeof(mt64_t));
  mt64_seed(g, seed);
  uint64_t word = 0;
  int left = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (left == 0) {
      word = mt64_next(g);
      left = 64;
    }
    bits[i] = (uint8_t)(word & 1);
    word >>= 1;
    --left;
  }
  free(g);
}

/* encode, codec.cpp:73-86: from state 0, no tail, B outputs per stage. */
int vdo_encode(int k, int b, const uint32_t* polys, const uint8_t* bits, int64_t n, uint8_t* coded) {
  if (validate_spec(k, b, polys)) return 1;
  uint32_t state = 0;
  for (int64_t t = 0; t < n; ++t) {
    const uint32_t u = bits[t] & 1;
    const uint32_t reg = (u << (k - 1)) | state;
    for (int i = 0; i < b; ++i) coded[t * b + i] = (uint8_t)(popcount32(polys[i] & reg) & 1);
    state = (u << (k - 2)) | (state >> 1);
  }
  return 0;
}

/* modulate_bpsk (channel.cpp:8-14) + awgn (:40-53) with NormalSampler
 * (:22-38): mt19937_64 standardized output into a Marsaglia polar pair. */
void vdo_awgn_bpsk(const uint8_t* coded, int64_t len, double sigma, uint64_t seed, double* rx) {
  if (sigma == 0.0) {
    for (int64_t i = 0; i < len; ++i) rx[i] = coded[i] ? -1.0 : 1.0;
    return;
  }
  mt64_t* g = malloc(sizeof(mt64_t));
  mt64_seed(g, seed);
  double cached = 0.0;
  int has_cached = 0;
  for (int64_t i = 0; i < len; ++i) {
    double z;
    if (has_cached) {
      has_cached = 0;
      z = cached;
    } else {
      for (;;) {
        const double u = 2.0 * ((double)(mt64_next(g) >> 11) * 0x1.0p-53) - 1.0;
        const double v = 2.0 * ((double)(mt64_next(g) >> 11) * 0x1.0p-53) - 1.0;
        const double s = u * u + v * v;
        if (s >= 1.0 || s == 0.0) continue;
        const double m = sqrt(-2.0 * log(s) / s);
        cached = v * m;
        has_cached = 1;
        z = u * m;
        break;
      }
    }
    const double sym = coded[i] ? -1.0 : 1.0;
    rx[i] = sym + sigma * z;
  }
  free(g);
}

static int gen_block(int k, int b, const uint32_t* polys, int64_t n, double sigma, uint64_t bits_seed,
                     uint64_t noise_seed, double* rx, uint8_t* sent) {
  if (validate_spec(k, b, polys)) return 1;
  vdo_random_bits(n, bits_seed, sent);
  uint8_t* coded = malloc((size_t)(n * b));
  vdo_encode(k, b, polys, sent, n, coded);
  vdo_awgn_bpsk(coded, n * b, sigma, noise_seed, rx);
  free(coded);
  return 0;
}

int vdo_gen_bench_block(int k, int b, const uint32_t* polys, int64_t n, double ebn0_db, uint64_t seed, double* rx,
                        uint8_t* sent) {
  /* berlab.cpp:138-142: base-rate sigma, seeds mix_seed(seed,1/2). */
  return gen_block(k, b, polys, n, vdo_sigma_from_ebn0(ebn0_db, 1.0 / b), vdo_mix_seed(seed, 1),
                   vdo_mix_seed(seed, 2), rx, sent);
}

int vdo_gen_sweep_block(int k, int b, const uint32_t* polys, int64_t n, double sigma, uint64_t block_seed,
                        double* rx, uint8_t* sent) {
  /* berlab.cpp:68-79 (identity puncture pattern) */
  return gen_block(k, b, polys, n, sigma, vdo_mix_seed(block_seed, 1), vdo_mix_seed(block_seed, 2), rx, sent);
}

void vdo_quantize_i8(const double* y, int64_t len, double scale, int8_t* q) {
  for (int64_t i = 0; i < len; ++i) {
    double v = nearbyint(scale * y[i]);
    if (v > 127.0) v = 127.0;
    if (v < -127.0) v = -127.0;
    q[i] = (int8_t)v;
  }
}

/* ---- puncturing -----------------------------------------------------------
 * mask: b x period, column-major (mask[col * b + row], reference
 * codec.hpp:15-21). validate = PuncturePattern::validate (codec.cpp:12-23). */
static int punct_validate(int b, int period, const uint8_t* mask) {
  if (b < 1 || period < 1 || !mask) return fail("puncture mask shape mismatch");
  for (int col = 0; col < period; ++col) {
    int kept = 0;
    for (int row = 0; row < b; ++row) kept += mask[col * b + row];
    if (kept == 0) return fail("puncture mask drops an entire stage");
  }
  return 0;
}

/* puncture (codec.cpp:88-103), on int8 soft values instead of bits: keeps
 * the mask-1 positions of a stage-major stream of n_stages stages. Writes
 * *out_len values. */
int vdo_puncture_i8(int b, int period, const uint8_t* mask, const int8_t* in, int64_t n_stages, int8_t* out,
                    int64_t* out_len) {
  if (punct_validate(b, period, mask)) return 1;
  int64_t idx = 0;
  for (int64_t t = 0; t < n_stages; ++t) {
    const int col = (int)(t % period);
    for (int row = 0; row < b; ++row) {
      if (mask[col * b + row]) out[idx++] = in[t * b + row];
    }
  }
  *out_len = idx;
  return 0;
}

/* depuncture (decoder.cpp:131-163): stage count from the punctured length
 * (throws "punctured length inconsistent with pattern"), then 0 at every
 * punctured position. out (may be NULL: count only) holds out_cap values. */
int vdo_depuncture_i8(int b, int period, const uint8_t* mask, const int8_t* in, int64_t len, int8_t* out,
                      int64_t out_cap, int64_t* stages_out) {
  if (punct_validate(b, period, mask)) return 1;
  int per_period = 0;
  for (int i = 0; i < b * period; ++i) per_period += mask[i];
  int64_t remaining = len;
  int64_t stages = (remaining / per_period) * period;
  remaining %= per_period;
  for (int col = 0; remaining > 0; ++col) {
    int kept = 0;
    if (col < period) {
      for (int row = 0; row < b; ++row) kept += mask[col * b + row];
    }
    if (col >= period || remaining < kept) return fail("punctured length inconsistent with pattern");
    remaining -= kept;
    ++stages;
  }
  *stages_out = stages;
  if (!out) return 0;
  if (stages * b > out_cap) return fail("output buffer too small");
  int64_t idx = 0;
  for (int64_t t = 0; t < stages; ++t) {
    const int col = (int)(t % period);
    for (int row = 0; row < b; ++row) out[t * b + row] = mask[col * b + row] ? in[idx++] : 0;
  }
  return 0;
}
