// C-ABI implementation (include/vitdec_b200.h): validation with the
// reference's exact messages, trellis construction, device dispatch, and the
// host-buffer streaming engine (H2D / decode / D2H overlapped per device,
// frames sharded across devices with no collective).
#include "vitdec_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <initializer_list>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "vd_common.cuh"
#include "vd_internal.h"

struct vd_code {
  int k = 0, b = 0, s = 0;
  std::vector<std::uint32_t> polys;
  std::vector<std::uint32_t> next, out, pred, in_out;
  bool complement_paired = false;
  mutable std::mutex mu;
  mutable std::map<int, std::uint32_t*> dev_in_out;  // device -> uploaded in_out table
  ~vd_code() {
    for (auto& kv : dev_in_out) {
      int prev = 0;
      if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(kv.first) == cudaSuccess) {
        cudaFree(kv.second);
        cudaSetDevice(prev);
      }
    }
  }
};

#ifndef VD_SERIAL_PARALLEL
#define VD_SERIAL_PARALLEL 1
#endif

namespace {

thread_local std::string g_err;

vd_status fail(vd_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

vd_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorInvalidSource && !vd::jit::last_log().empty()) msg += " (" + vd::jit::last_log() + ")";
  return fail(VD_ECUDA, msg);
}

#define VD_CUDA(call, what)                         \
  do {                                              \
    const cudaError_t vd_e_ = (call);               \
    if (vd_e_ != cudaSuccess) return cuda_fail(vd_e_, what); \
  } while (0)

// Trellis validation: messages of reference trellis.cpp:38-53.
vd_status validate_spec(int k, int b, const std::uint32_t* polys) {
  if (k < 2) return fail(VD_EINVAL, "constraint length must be >= 2");
  if (b < 2) return fail(VD_EINVAL, "need at least 2 outputs per bit");
  if (!polys) return fail(VD_EINVAL, "polynomial count must equal B");
  if (k > 16) return fail(VD_EINVAL, "constraint length too large");
  const std::uint32_t mask = (1u << k) - 1;
  for (int i = 0; i < b; ++i) {
    if (polys[i] == 0) return fail(VD_EINVAL, "zero generator polynomial");
    if ((polys[i] & ~mask) != 0) return fail(VD_EINVAL, "generator polynomial wider than K bits");
  }
  return VD_OK;
}

// FrameConfig::validate, reference decoder.cpp:10-20.
vd_status validate_cfg(const vd_frame_cfg* cfg, int period) {
  if (!cfg) return fail(VD_EINVAL, "null frame config");
  if (cfg->f < 1) return fail(VD_EINVAL, "frame size f must be >= 1");
  if (cfg->v1 < 0 || cfg->v2 < 0) return fail(VD_EINVAL, "overlaps must be >= 0");
  if (cfg->f0 < 0 || cfg->f0 > cfg->f) return fail(VD_EINVAL, "f0 must be in [0, f]");
  if (period > 1 && (cfg->f % period || cfg->v1 % period || cfg->v2 % period)) {
    return fail(VD_EINVAL, "f, v1 and v2 must be multiples of the puncture period");
  }
  if (cfg->start != VD_TB_STORED_MAX && cfg->start != VD_TB_RANDOM) {
    return fail(VD_EINVAL, "unknown traceback start");
  }
  return VD_OK;
}

std::int64_t num_frames(const vd_frame_cfg* cfg, std::int64_t n) { return (n + cfg->f - 1) / cfg->f; }

// Frames per output-word-aligned unit: L*f is a multiple of 32.
std::int64_t align_unit(int f) {
  int g = 32;
  int x = f;
  while (x) {
    const int t = g % x;
    g = x;
    x = t;
  }
  return 32 / g;
}

vd_status check_gpu_envelope(const vd_code* code) {
  if (code->k > vd::kMaxK) return fail(VD_EUNSUPPORTED, "GPU decoder supports K <= 16");
  if (code->b > 8) return fail(VD_EUNSUPPORTED, "GPU decoder supports B <= 8");
  return VD_OK;
}

// ---- puncturing (reference codec.hpp:13-33, codec.cpp:12-23, decoder.cpp:131-163)
struct PunctPlan {
  int b = 0, period = 0, kept = 0;  // kept = kept_per_period()
  std::vector<std::int64_t> srank;  // kept bytes of columns [0, col): period + 1 entries
  std::vector<std::int16_t> rank;   // per cell (col * b + row): kept index in the period, or -1
  // absolute offset in the punctured stream of stage t's first kept byte
  std::int64_t off(std::int64_t t) const { return (t / period) * kept + srank[t % period]; }
};

// PuncturePattern::validate (codec.cpp:12-23) plus the GPU envelope.
vd_status make_punct(const vd_puncture* pat, PunctPlan* pp) {
  if (!pat || !pat->mask || pat->b < 1 || pat->period < 1) return fail(VD_EINVAL, "puncture mask shape mismatch");
  if (static_cast<std::int64_t>(pat->b) * pat->period > vd::kMaxPunctureCells) {
    return fail(VD_EUNSUPPORTED, "GPU depuncture supports period * B <= 1024");
  }
  pp->b = pat->b;
  pp->period = pat->period;
  pp->kept = 0;
  pp->srank.assign(static_cast<std::size_t>(pat->period) + 1, 0);
  pp->rank.assign(static_cast<std::size_t>(pat->period) * pat->b, -1);
  for (int col = 0; col < pat->period; ++col) {
    int kept = 0;
    for (int row = 0; row < pat->b; ++row) {
      const std::uint8_t m = pat->mask[col * pat->b + row];
      if (m > 1) return fail(VD_EINVAL, "puncture mask must be 0/1");
      if (m) pp->rank[col * pat->b + row] = static_cast<std::int16_t>(pp->kept + kept++);
    }
    if (kept == 0) return fail(VD_EINVAL, "puncture mask drops an entire stage");
    pp->kept += kept;
    pp->srank[col + 1] = pp->kept;
  }
  return VD_OK;
}

// Patterns with a fused-depuncture fast-kernel instantiation (vd_fast.cuh
// PunctR23 / PunctR34): 23 = "11;10", 34 = "110;101"; 0 = none.
int punct_pattern_id(const PunctPlan& pp) {
  if (pp.b != 2) return 0;
  auto is = [&](int period, std::initializer_list<int> kept_cells) {
    if (pp.period != period) return false;
    std::vector<int> want(static_cast<std::size_t>(period) * 2, -1);
    int r = 0;
    for (int q = 0; q < period * 2; ++q) {
      const bool k = std::find(kept_cells.begin(), kept_cells.end(), q) != kept_cells.end();
      if (k) want[q] = r++;
    }
    for (int q = 0; q < period * 2; ++q) {
      if ((pp.rank[q] >= 0) != (want[q] >= 0)) return false;
    }
    return true;
  };
  if (is(2, {0, 1, 2})) return 23;     // col0 rows 0,1; col1 row 0
  if (is(3, {0, 1, 2, 5})) return 34;  // col0 rows 0,1; col1 row 0; col2 row 1
  return 0;
}

// Stage count of a punctured stream (decoder.cpp:141-152).
vd_status punct_stages(const PunctPlan& pp, std::int64_t len, std::int64_t* stages) {
  if (len < 0) return fail(VD_EINVAL, "punctured length inconsistent with pattern");
  std::int64_t st = (len / pp.kept) * pp.period;
  std::int64_t rem = len % pp.kept;
  for (int col = 0; rem > 0; ++col) {
    const std::int64_t ck = pp.srank[col + 1] - pp.srank[col];
    if (col >= pp.period || rem < ck) return fail(VD_EINVAL, "punctured length inconsistent with pattern");
    rem -= ck;
    ++st;
  }
  *stages = st;
  return VD_OK;
}

// Depuncture stages [t0, t0 + n) from `in` (= the punctured stream at offset off(t0)).
vd_status launch_depuncture(const PunctPlan& pp, const std::int8_t* in, std::int64_t t0, std::int64_t n,
                            std::int8_t* out, cudaStream_t s) {
  vd::DepunctureLaunch d;
  d.in = in;
  d.in0 = pp.off(t0);
  d.out = out;
  d.t0 = t0;
  d.n = n;
  d.b = pp.b;
  d.period = pp.period;
  d.kept = pp.kept;
  d.in_len = pp.off(t0 + n) - d.in0;
  // unit = U whole periods, >= 1 KiB of output; U * period * b a multiple of
  // 16 and U * kept a multiple of 4 (unit-invariant byte alignment); tile =
  // tu units, ~32 KiB of output per shared-memory staging round
  const int pb = pp.period * pp.b;
  int unit = 16;
  for (int x = pb; x % 2 == 0 && unit > 1; x /= 2) unit /= 2;  // 16 / gcd(pb, 16)
  int unit_in = 4;
  for (int x = pp.kept; x % 2 == 0 && unit_in > 1; x /= 2) unit_in /= 2;  // 4 / gcd(kept, 4)
  unit = std::max(unit, unit_in);                                          // both powers of two
  d.unit_periods = std::max(unit, (1024 / pb + unit - 1) / unit * unit);
  d.unit_bytes = d.unit_periods * pb;
  d.unit_in = d.unit_periods * pp.kept;
  d.tu = std::max(1, 32768 / d.unit_bytes);
  std::copy(pp.rank.begin(), pp.rank.end(), d.rank);
  const cudaError_t e = vd::launch_depuncture_i8(d, s);
  if (e != cudaSuccess) return cuda_fail(e, "depuncture kernel");
  return VD_OK;
}

vd_status device_table(const vd_code* code, int device, const std::uint32_t** out) {
  std::lock_guard<std::mutex> lk(code->mu);
  auto it = code->dev_in_out.find(device);
  if (it != code->dev_in_out.end()) {
    *out = it->second;
    return VD_OK;
  }
  std::uint32_t* d = nullptr;
  VD_CUDA(cudaMalloc(&d, sizeof(std::uint32_t) * code->in_out.size()), "cudaMalloc(in_out)");
  VD_CUDA(cudaMemcpy(d, code->in_out.data(), sizeof(std::uint32_t) * code->in_out.size(), cudaMemcpyHostToDevice),
          "upload in_out");
  code->dev_in_out[device] = d;
  *out = d;
  return VD_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

vd_status resolve_device(int32_t device, int* out) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(VD_ECUDA, "no CUDA device available (the decoder has no CPU fallback)");
  }
  if (device < 0) {
    VD_CUDA(cudaGetDevice(out), "cudaGetDevice");
    return VD_OK;
  }
  if (device >= count) return fail(VD_EINVAL, "device index out of range");
  *out = device;
  return VD_OK;
}

template <typename T>
vd_status decode_device(const vd_code* code, const vd_frame_cfg* cfg, std::int64_t n, const T* llr,
                        std::int64_t llr_stage0, std::int64_t fb, std::int64_t fe, std::uint32_t* out,
                        std::int64_t out_stage0, void* sigma, std::int32_t device, void* stream) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (n < 1) return fail(VD_EINVAL, "empty llr block");
  if (vd_status st = check_gpu_envelope(code)) return st;
  const std::int64_t nf = num_frames(cfg, n);
  if (fb < 0 || fe > nf || fb > fe) return fail(VD_EINVAL, "frame range out of bounds");
  if (out_stage0 % 32 != 0) return fail(VD_EINVAL, "out_stage0 must be a multiple of 32");
  if (fb == fe) return VD_OK;
  if (!llr || !out) return fail(VD_EINVAL, "null buffer");
  const vd::FrameGeom g0(fb, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
  const vd::FrameGeom g1(fe - 1, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
  if (llr_stage0 > g0.beg) return fail(VD_EINVAL, "llr window does not cover the frames' warm-up stages");
  if (out_stage0 > g0.out_lo) return fail(VD_EINVAL, "output window starts after the first frame");

  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  const std::uint32_t* in_out = nullptr;
  if (vd_status st = device_table(code, dev, &in_out)) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  VD_CUDA(vd::retain_async_pool(), "memory pool");
  const std::int64_t w0 = (g0.out_lo - out_stage0) / 32;
  const std::int64_t w1 = (g1.out_hi - out_stage0 + 31) / 32;

  vd::DecodeLaunch p;
  p.k = code->k;
  p.b = code->b;
  p.s = code->s;
  p.f = cfg->f;
  p.v1 = cfg->v1;
  p.v2 = cfg->v2;
  p.f0 = cfg->f0;
  p.start = cfg->start;
  p.seed = cfg->seed;
  p.n = n;
  p.frame_begin = fb;
  p.frame_end = fe;
  p.llr = llr;
  p.llr_stage0 = llr_stage0;
  p.out = out;
  p.out_stage0 = out_stage0;
  p.sigma = sigma;
  p.in_out = in_out;
  for (int i = 0; i < code->b && i < 8; ++i) p.polys[i] = code->polys[i];
  p.complement_paired = code->complement_paired;

  // Zero the output words the frames touch (kernels OR bits into them),
  // unless the launch writes every word whole.
  bool whole = false;
  if constexpr (sizeof(T) == 1) whole = vd::fast_output_whole_words(p);
  if (!whole) VD_CUDA(cudaMemsetAsync(out + w0, 0, sizeof(std::uint32_t) * (w1 - w0), s), "zero output");

  cudaError_t e;
  if constexpr (sizeof(T) == 1) {
    if (vd::fast_path_supported(p)) {
      e = vd::launch_fast_i8(p, s);
    } else if (VD_SERIAL_PARALLEL && vd::serial_parallel_supported(p)) {
      e = vd::launch_serial_parallel_i8(p, s);
    } else {
      e = vd::launch_generic_i8(p, s);
    }
  } else {
    e = vd::launch_generic_f64(p, s);
  }
  if (e == cudaErrorInvalidValue) return fail(VD_EUNSUPPORTED, "frame configuration exceeds the GPU kernel's shared-memory envelope");
  if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
  return VD_OK;
}

// ---- batched independent blocks -------------------------------------------
// Every block runs its own framed decode (own frame grid, clipped at both of
// its ends, block-local random-start salt), as reference run_ber_sweep calls
// framed_decode once per block (berlab.cpp:63-88) — but all blocks go to the
// device in one fast-kernel launch plus one generic launch for the clipped
// edge frames of every block.

void batch_stats(const vd_frame_cfg* cfg, std::int32_t nblocks, const std::int64_t* lens, vd_stats* st) {
  st->frames = st->stages = st->tracebacks = 0;
  std::int64_t last_len = -1;
  vd_stats b{};
  for (std::int32_t j = 0; j < nblocks; ++j) {
    if (lens[j] != last_len) {  // BER-sweep batches repeat one block length
      vd_frame_stats(cfg, lens[j], &b);
      last_len = lens[j];
    }
    st->frames += b.frames;
    st->stages += b.stages;
    st->tracebacks += b.tracebacks;
  }
}

template <typename T>
vd_status decode_batch_device(const vd_code* code, const vd_frame_cfg* cfg, std::int32_t nblocks,
                              const std::int64_t* lens, const T* llr, std::uint32_t* out, vd_stats* stats,
                              std::int32_t device, void* stream) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (nblocks < 1 || !lens) return fail(VD_EINVAL, "batch needs at least one block");
  for (std::int32_t j = 0; j < nblocks; ++j) {
    if (lens[j] < 1) return fail(VD_EINVAL, "empty llr block");  // reference decoder.cpp:92-97
  }
  if (vd_status st = check_gpu_envelope(code)) return st;
  if (!llr || !out) return fail(VD_EINVAL, "null buffer");
  if (stats) batch_stats(cfg, nblocks, lens, stats);

  // Block tables: stage and frame prefixes, fast-kernel interior range per
  // block, and the list of remaining (edge) frames.
  const int f = cfg->f, v1 = cfg->v1, v2 = cfg->v2, B = code->b;
  const std::int64_t L = static_cast<std::int64_t>(f) + v1 + v2;
  std::vector<std::int64_t> bstage(nblocks + 1, 0), bframe(nblocks + 1, 0);
  for (std::int32_t j = 0; j < nblocks; ++j) {
    bstage[j + 1] = bstage[j] + lens[j];
    bframe[j + 1] = bframe[j] + num_frames(cfg, lens[j]);
  }
  const std::int64_t n_total = bstage[nblocks], nf_total = bframe[nblocks];

  vd::DecodeLaunch p;
  p.k = code->k;
  p.b = code->b;
  p.s = code->s;
  p.f = f;
  p.v1 = v1;
  p.v2 = v2;
  p.f0 = cfg->f0;
  p.start = cfg->start;
  p.seed = cfg->seed;
  p.n = n_total;
  p.llr = llr;
  p.out = out;
  for (int i = 0; i < code->b && i < 8; ++i) p.polys[i] = code->polys[i];
  p.complement_paired = code->complement_paired;
  // Does the fast kernel take this code/config at all? (probe on one long stream)
  bool fast = false;
  if constexpr (sizeof(T) == 1) {
    vd::DecodeLaunch probe = p;
    probe.n = std::max<std::int64_t>(n_total, 64 * L);
    probe.frame_begin = 0;
    probe.frame_end = num_frames(cfg, probe.n);
    fast = vd::fast_path_supported(probe);
  }
  std::vector<std::int32_t> ilo(nblocks, 0), ihi(nblocks, 0);
  std::vector<std::int64_t> edges;
  std::int64_t safe = -1, interior = 0;
  // Edge frames the fast kernel can still take (int8 path): HEAD frames
  // (window clipped at the block start, full right window) read a zero-padded
  // copy of their block head — all-zero branch metrics keep sigma = 0 until
  // stage 0 — and TAIL frames with a full output but a clipped right overlap
  // v2' < v2 are exactly frames of configuration (f, v1, v2') (one traceback
  // per frame: the start stage is the window end either way), one launch per
  // distinct v2'. Everything else goes to the generic kernel.
  const std::int64_t head_end = (v1 + f - 1) / f;
  const bool one_tb = cfg->f0 == 0 || cfg->f0 >= f;
  // test / A-B hooks: VITDEC_BATCH_EDGES=generic keeps every edge frame on the generic kernel
  const char* env_edges = std::getenv("VITDEC_BATCH_EDGES");
  const int edge_mode = !env_edges ? 3 : std::strcmp(env_edges, "generic") == 0 ? 0
                        : std::strcmp(env_edges, "heads") == 0 ? 1 : std::strcmp(env_edges, "tails") == 0 ? 2 : 3;
  std::vector<std::int64_t> heads;
  std::map<int, std::vector<std::int64_t>> tails;  // v2' -> global frame ids
  // BER-sweep batches repeat one block length: the per-block classification is
  // memoised per length (valid for aligned blocks away from the stream end).
  struct Memo {
    std::int64_t len = -1, lo = 0, hi = 0;
    std::vector<std::pair<std::int64_t, int>> edge;  // (m, kind): 0 generic, 1 head, 2 + v2' tail
  } memo;
  heads.reserve(static_cast<std::size_t>(nblocks));
  std::vector<std::int64_t>* last_tail = nullptr;
  int last_key = -1;
  auto classify = [&](std::int32_t j, std::int64_t lo, std::int64_t hi, bool aligned,
                      std::vector<std::pair<std::int64_t, int>>& outv) {
    const std::int64_t nfj = bframe[j + 1] - bframe[j];
    for (std::int64_t m = 0; m < nfj; ++m) {
      if (m == lo && hi > lo) m = hi;  // skip the interior run (the fast kernel's)
      if (m >= nfj) break;
      int kind = 0;
      if ((edge_mode & 1) && aligned && m < head_end && m * f + f + v2 <= lens[j]) {
        kind = 1;
      } else if ((edge_mode & 2) && aligned && one_tb && m >= head_end && m * f + f <= lens[j] &&
                 m * f + f + v2 > lens[j] && f + v1 + (lens[j] - m * f - f) >= 16 &&
                 bstage[j] + lens[j] + vd::kPfSlackStages <= n_total) {
        kind = 2 + static_cast<int>(lens[j] - m * f - f);
      }
      outv.emplace_back(m, kind);
    }
  };
  std::vector<std::pair<std::int64_t, int>> scratch_edges;
  for (std::int32_t j = 0; j < nblocks; ++j) {
    const bool aligned = fast && (bstage[j] * B) % 4 == 0;
    // memo valid: same length, aligned, and window + slack of every frame inside the stream
    const bool regular = aligned && bstage[j] + lens[j] + L + vd::kPfSlackStages + f <= n_total;
    std::int64_t lo = 0, hi = 0;
    const std::vector<std::pair<std::int64_t, int>>* ev;
    if (regular && memo.len == lens[j]) {
      lo = memo.lo;
      hi = memo.hi;
      ev = &memo.edge;
    } else {
      if (aligned) {
        lo = (v1 + f - 1) / f;                                        // m*f >= v1
        hi = lens[j] - f - v2 >= 0 ? (lens[j] - f - v2) / f + 1 : 0;  // m*f + f + v2 <= n_j
        // window + the fast kernel's read slack inside the whole stream
        const std::int64_t room = n_total - bstage[j] + v1 - L - vd::kPfSlackStages;
        hi = std::min(hi, room >= 0 ? room / f + 1 : 0);
        hi = std::max(hi, lo);
      }
      scratch_edges.clear();
      classify(j, lo, hi, aligned, scratch_edges);
      if (regular) {
        memo.len = lens[j];
        memo.lo = lo;
        memo.hi = hi;
        memo.edge = scratch_edges;
        ev = &memo.edge;
      } else {
        ev = &scratch_edges;
      }
    }
    ilo[j] = static_cast<std::int32_t>(lo);
    ihi[j] = static_cast<std::int32_t>(hi);
    if (hi > lo && safe < 0) safe = bstage[j] + lo * f - v1;
    interior += hi - lo;
    for (const auto& e : *ev) {
      const std::int64_t id = bframe[j] + e.first;
      if (e.second == 0) {
        edges.push_back(id);
      } else if (e.second == 1) {
        heads.push_back(id);
      } else {
        const int key = e.second - 2;
        if (key != last_key) {
          last_tail = &tails[key];
          last_key = key;
        }
        last_tail->push_back(id);
      }
    }
  }

  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  const std::uint32_t* in_out = nullptr;
  if (vd_status st = device_table(code, dev, &in_out)) return st;
  p.in_out = in_out;
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  // Stream-ordered scratch for the tables (freed after the launches).
  const std::size_t nb1 = static_cast<std::size_t>(nblocks) + 1;
  // frame lists: generic edges, then heads, then every tail class
  std::vector<std::int64_t> lists = edges;
  const std::size_t heads_off = lists.size();
  lists.insert(lists.end(), heads.begin(), heads.end());
  std::vector<std::pair<int, std::size_t>> tail_off;  // (v2', offset)
  for (auto& kv : tails) {
    tail_off.emplace_back(kv.first, lists.size());
    lists.insert(lists.end(), kv.second.begin(), kv.second.end());
  }
  const std::size_t bytes = sizeof(std::int64_t) * (2 * nb1 + lists.size()) + sizeof(std::int32_t) * 2 * nb1;
  // pinned staging (per host thread and device, grows) so the table upload is
  // a true async copy; the event is created on the device whose stream records it
  struct BatchStaging {
    unsigned char* pinned = nullptr;
    std::size_t cap = 0;
    cudaEvent_t done = nullptr;  // last upload out of the staging buffer
  };
  thread_local std::map<int, BatchStaging> staging;
  BatchStaging& bs = staging[dev];
  unsigned char*& pinned = bs.pinned;
  std::size_t& pinned_cap = bs.cap;
  cudaEvent_t& pinned_done = bs.done;
  if (pinned_done) VD_CUDA(cudaEventSynchronize(pinned_done), "batch table staging");
  if (pinned_cap < bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_cap = 0;
    VD_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned), bytes), "cudaMallocHost(batch tables)");
    pinned_cap = bytes;
  }
  unsigned char* host_p = pinned;
  std::memcpy(host_p, bstage.data(), sizeof(std::int64_t) * nb1);
  std::memcpy(host_p + sizeof(std::int64_t) * nb1, bframe.data(), sizeof(std::int64_t) * nb1);
  std::memcpy(host_p + sizeof(std::int64_t) * 2 * nb1, lists.data(), sizeof(std::int64_t) * lists.size());
  const std::size_t i32_off = sizeof(std::int64_t) * (2 * nb1 + lists.size());
  std::memcpy(host_p + i32_off, ilo.data(), sizeof(std::int32_t) * nblocks);
  std::memcpy(host_p + i32_off + sizeof(std::int32_t) * nb1, ihi.data(), sizeof(std::int32_t) * nblocks);
  unsigned char* dscratch = nullptr;
  VD_CUDA(vd::retain_async_pool(), "memory pool");
  VD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dscratch), bytes, s), "cudaMallocAsync(batch tables)");
  VD_CUDA(cudaMemcpyAsync(dscratch, host_p, bytes, cudaMemcpyHostToDevice, s), "upload batch tables");
  if (!pinned_done) VD_CUDA(cudaEventCreateWithFlags(&pinned_done, cudaEventDisableTiming), "cudaEventCreate");
  VD_CUDA(cudaEventRecord(pinned_done, s), "cudaEventRecord");
  p.nblocks = nblocks;
  p.blk_stage = reinterpret_cast<const std::int64_t*>(dscratch);
  p.blk_frame = p.blk_stage + nb1;
  p.blk_ilo = reinterpret_cast<const std::int32_t*>(dscratch + i32_off);
  p.blk_ihi = p.blk_ilo + nb1;
  const std::int64_t* dedges = p.blk_stage + 2 * nb1;

  VD_CUDA(cudaMemsetAsync(out, 0, sizeof(std::uint32_t) * ((n_total + 31) / 32), s), "zero output");
  cudaError_t e = cudaSuccess;
  bool fast_launched = false;
  std::int64_t* extra_list = nullptr;
  std::int8_t* head_buf = nullptr;
  if (fast && interior > 0) {
    vd::DecodeLaunch q = p;
    q.frame_begin = 0;
    q.frame_end = nf_total;
    q.safe_stage = safe;
    if (vd::fast_path_supported(q)) {
      e = vd::launch_fast_i8(q, s);
      fast_launched = true;
    }
  }
  // head and tail classes on the fast kernel (frame-list launches)
  std::vector<std::int64_t> back_to_generic;
  if constexpr (sizeof(T) == 1) {
    if (e == cudaSuccess && fast_launched && !heads.empty()) {
      // 4-byte aligned block heads, each followed by the fast kernel's read slack
      const std::int64_t pitch = (v1 + head_end * f + v2 + vd::kPfSlackStages + 3) & ~std::int64_t(3);
      e = cudaMallocAsync(reinterpret_cast<void**>(&head_buf), static_cast<std::size_t>(pitch) * B * nblocks + 16, s);
      if (e == cudaSuccess)
        e = vd::launch_head_gather(reinterpret_cast<const std::int8_t*>(llr), p.blk_stage, nblocks, B, v1, pitch,
                                   head_end * f + v2, head_buf, s);
      vd::DecodeLaunch q = p;
      q.frame_list = dedges + heads_off;
      q.frame_begin = 0;
      q.frame_end = static_cast<std::int64_t>(heads.size());
      q.safe_stage = safe;
      q.llr_head = head_buf;
      q.head_pitch = pitch;
      if (e == cudaSuccess) {
        if (vd::fast_path_supported(q)) {
          e = vd::launch_fast_i8(q, s);
        } else {
          back_to_generic.insert(back_to_generic.end(), heads.begin(), heads.end());
        }
      }
    } else if (!heads.empty()) {
      back_to_generic.insert(back_to_generic.end(), heads.begin(), heads.end());
    }
    for (const auto& to : tail_off) {
      const std::vector<std::int64_t>& lst = tails[to.first];
      vd::DecodeLaunch q = p;
      q.v2 = to.first;
      q.frame_list = dedges + to.second;
      q.frame_begin = 0;
      q.frame_end = static_cast<std::int64_t>(lst.size());
      q.safe_stage = safe;
      if (e == cudaSuccess && fast_launched && vd::fast_path_supported(q)) {
        e = vd::launch_fast_i8(q, s);
      } else {
        back_to_generic.insert(back_to_generic.end(), lst.begin(), lst.end());
      }
    }
  }
  if (e == cudaSuccess) {
    vd::DecodeLaunch q = p;
    q.frame_begin = 0;
    if (fast_launched && back_to_generic.empty()) {
      q.frame_list = dedges;
      q.frame_end = static_cast<std::int64_t>(edges.size());
    } else if (fast_launched) {
      // rare: a head / tail class the fast kernel declined; decode the whole
      // remaining list (edges + declined frames) with the generic kernel
      std::vector<std::int64_t> all = edges;
      all.insert(all.end(), back_to_generic.begin(), back_to_generic.end());
      std::int64_t* dl = nullptr;
      VD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dl), sizeof(std::int64_t) * all.size(), s), "cudaMallocAsync");
      VD_CUDA(cudaMemcpyAsync(dl, all.data(), sizeof(std::int64_t) * all.size(), cudaMemcpyHostToDevice, s), "H2D");
      q.frame_list = dl;
      q.frame_end = static_cast<std::int64_t>(all.size());
      extra_list = dl;
    } else {
      q.frame_end = nf_total;
    }
    if (q.frame_end > 0) {
      if constexpr (sizeof(T) == 1) {
        e = vd::launch_generic_i8(q, s);
      } else {
        e = vd::launch_generic_f64(q, s);
      }
    }
  }
  if (extra_list) cudaFreeAsync(extra_list, s);
  if (head_buf) cudaFreeAsync(head_buf, s);
  const cudaError_t ef = cudaFreeAsync(dscratch, s);
  if (e == cudaErrorInvalidValue) return fail(VD_EUNSUPPORTED, "frame configuration exceeds the GPU kernel's shared-memory envelope");
  if (e != cudaSuccess) return cuda_fail(e, "batched decode launch");
  if (ef != cudaSuccess) return cuda_fail(ef, "cudaFreeAsync(batch tables)");
  return VD_OK;
}

// ---- host-buffer streaming engine ----------------------------------------

struct DevCtx {
  cudaStream_t st[2] = {nullptr, nullptr};
  void* llr[2] = {nullptr, nullptr};
  std::size_t llr_cap[2] = {0, 0};
  std::uint32_t* out[2] = {nullptr, nullptr};
  std::size_t out_cap[2] = {0, 0};
  void* pun[2] = {nullptr, nullptr};  // punctured-stream staging (depuncture input)
  std::size_t pun_cap[2] = {0, 0};
  // pinned host staging for pageable caller buffers (input chunks / output words)
  void* hin[2] = {nullptr, nullptr};
  std::size_t hin_cap[2] = {0, 0};
  void* hout[2] = {nullptr, nullptr};
  std::size_t hout_cap[2] = {0, 0};
  cudaEvent_t hin_free[2] = {nullptr, nullptr}, hout_ready[2] = {nullptr, nullptr};
  bool hin_used[2] = {false, false}, hout_pending[2] = {false, false};
  std::uint32_t* pend_dst[2] = {nullptr, nullptr};
  std::size_t pend_bytes[2] = {0, 0};
};

struct ThreadCtx {
  std::map<int, DevCtx> devs;
  ~ThreadCtx() {
    for (auto& kv : devs) {
      if (cudaSetDevice(kv.first) != cudaSuccess) continue;
      for (int i = 0; i < 2; ++i) {
        if (kv.second.llr[i]) cudaFree(kv.second.llr[i]);
        if (kv.second.out[i]) cudaFree(kv.second.out[i]);
        if (kv.second.pun[i]) cudaFree(kv.second.pun[i]);
        if (kv.second.hin[i]) cudaFreeHost(kv.second.hin[i]);
        if (kv.second.hout[i]) cudaFreeHost(kv.second.hout[i]);
        if (kv.second.hin_free[i]) cudaEventDestroy(kv.second.hin_free[i]);
        if (kv.second.hout_ready[i]) cudaEventDestroy(kv.second.hout_ready[i]);
        if (kv.second.st[i]) cudaStreamDestroy(kv.second.st[i]);
      }
    }
  }
};

thread_local ThreadCtx tl_ctx;

vd_status ensure(void** p, std::size_t* cap, std::size_t bytes) {
  if (*cap >= bytes) return VD_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  VD_CUDA(cudaMalloc(p, bytes), "cudaMalloc(stream buffer)");
  *cap = bytes;
  return VD_OK;
}

struct Chunk {
  std::int64_t f0, f1;  // frame range
};

// Page-locked host memory reaches full PCIe rate with async copies; pageable
// caller buffers (numpy arrays, std::vector, Eigen blocks) are staged through
// per-(thread, device) pinned buffers, the host copy split over a few threads.
bool host_pinned(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Persistent host-copy workers (one pool per process, shared by every calling
// thread): staging copies of pageable buffers are split over up to
// VITDEC_COPY_THREADS threads (default: all hardware threads, at most 16)
// without a thread create / join per chunk.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();  // never destroyed: workers park on the condition variable at exit
    return *pool;
  }
  int threads() const { return nt_; }
  // Runs fn(0..parts-1): part 0 on the caller, the rest on the workers.
  void run(int parts, const std::function<void(int)>& fn) {
    struct Done {
      std::mutex mu;
      std::condition_variable cv;
      int left;
    } done;
    done.left = parts - 1;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int i = 1; i < parts; ++i) {
        q_.emplace_back([&fn, &done, i] {
          fn(i);
          std::lock_guard<std::mutex> dl(done.mu);
          if (--done.left == 0) done.cv.notify_one();
        });
      }
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> dl(done.mu);
    done.cv.wait(dl, [&] { return done.left == 0; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int nt = static_cast<int>(std::min(16u, hw));
    if (const char* e = std::getenv("VITDEC_COPY_THREADS")) nt = std::max(1, std::atoi(e));
    nt_ = 1;
    for (int i = 1; i < nt; ++i) {
      try {
        std::thread([this] { work(); }).detach();
        ++nt_;
      } catch (...) {  // no more threads: copy with the ones we have (never throw across the C-ABI)
        break;
      }
    }
  }
  void work() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty(); });
        job = std::move(q_.front());
        q_.pop_front();
      }
      job();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  int nt_ = 1;
};

void parallel_memcpy(void* dst, const void* src, std::size_t bytes) {
  constexpr std::size_t kMinPart = std::size_t{2} << 20;  // smaller copies: a pool hand-off costs more than it saves
  CopyPool& pool = CopyPool::get();
  const int nt = static_cast<int>(std::min<std::size_t>(pool.threads(), std::max<std::size_t>(1, bytes / kMinPart)));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const std::size_t part = (bytes / nt + 63) & ~std::size_t{63};
  pool.run(nt, [=](int i) {
    const std::size_t lo = static_cast<std::size_t>(i) * part;
    if (lo < bytes) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, std::min(part, bytes - lo));
  });
}

vd_status ensure_host(void** p, std::size_t* cap, std::size_t bytes) {
  if (*cap >= bytes) return VD_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  VD_CUDA(cudaMallocHost(p, bytes), "cudaMallocHost(staging)");
  *cap = bytes;
  return VD_OK;
}

// pp != nullptr (int8 only): `llr` is the PUNCTURED stream of pattern pp
// covering n stages; each chunk's punctured bytes are copied and expanded on
// the device (depuncture kernel) right before its decode.
// llr4 != nullptr (int8 only): the stream is in the 4-bit wire format
// (element i in nibble i of llr4, low nibble first); each chunk's bytes are
// copied and widened to int8 on the device (vd_wire.cu) before its decode.
template <typename T>
vd_status decode_host(const vd_code* code, const vd_frame_cfg* cfg, const T* llr, std::int64_t n,
                      std::uint32_t* out_packed, vd_stats* stats, const vd_exec* exec,
                      const PunctPlan* pp = nullptr, const std::uint8_t* llr4 = nullptr) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (n < 1) return fail(VD_EINVAL, "empty llr block");
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (stats) {
    if (vd_status st = vd_frame_stats(cfg, n, stats)) return st;
  }
  if (vd_status st = check_gpu_envelope(code)) return st;
  if (!llr || !out_packed) return fail(VD_EINVAL, "null buffer");

  // Devices.
  std::vector<int> devices;
  {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      return fail(VD_ECUDA, "no CUDA device available (the decoder has no CPU fallback)");
    }
    const int want = (exec && exec->num_devices > 0) ? exec->num_devices : 0;
    if (want == 0) {
      int cur = 0;
      VD_CUDA(cudaGetDevice(&cur), "cudaGetDevice");
      devices.push_back(cur);
    } else {
      for (int i = 0; i < want; ++i) {
        const int d = exec->devices ? exec->devices[i] : i;
        if (d < 0 || d >= count) return fail(VD_EINVAL, "device index out of range");
        devices.push_back(d);
      }
    }
  }
  const int nd = static_cast<int>(devices.size());
  std::vector<std::int64_t> first(nd + 1);
  if (vd_status st = vd_partition_frames(cfg, n, nd, first.data())) return st;

  // Chunk plan: whole output-word-aligned units of frames per chunk.
  const std::int64_t unit = align_unit(cfg->f);
  std::int64_t chunk_stages = (exec && exec->chunk_stages > 0) ? exec->chunk_stages : (std::int64_t{1} << 24);
  std::int64_t chunk_frames = std::max<std::int64_t>(unit, (chunk_stages / cfg->f) / unit * unit);
  std::vector<std::vector<Chunk>> plan(nd);
  std::size_t max_chunks = 0;
  for (int d = 0; d < nd; ++d) {
    for (std::int64_t c = first[d]; c < first[d + 1]; c += chunk_frames) {
      plan[d].push_back({c, std::min(c + chunk_frames, first[d + 1])});
    }
    max_chunks = std::max(max_chunks, plan[d].size());
  }
  // Buffer sizes per device.
  const std::int64_t max_window = std::min<std::int64_t>(chunk_frames * cfg->f + cfg->v1 + cfg->v2, n);
  const std::size_t llr_bytes = sizeof(T) * static_cast<std::size_t>(max_window) * code->b;
  const std::int64_t max_out = std::min<std::int64_t>(chunk_frames * cfg->f, n);  // f >= n: one clipped frame
  const std::size_t out_bytes = sizeof(std::uint32_t) * static_cast<std::size_t>((max_out + 31) / 32 + 1);

  for (int d = 0; d < nd; ++d) {
    if (plan[d].empty()) continue;
    DeviceGuard guard(devices[d]);
    DevCtx& ctx = tl_ctx.devs[devices[d]];
    for (int i = 0; i < 2; ++i) {
      if (!ctx.st[i]) VD_CUDA(cudaStreamCreateWithFlags(&ctx.st[i], cudaStreamNonBlocking), "cudaStreamCreate");
      if (vd_status st = ensure(&ctx.llr[i], &ctx.llr_cap[i], llr_bytes)) return st;
      if (pp || llr4) {
        if (vd_status st = ensure(&ctx.pun[i], &ctx.pun_cap[i], llr_bytes)) return st;
      }
      void* o = ctx.out[i];
      if (vd_status st = ensure(&o, &ctx.out_cap[i], out_bytes)) return st;
      ctx.out[i] = static_cast<std::uint32_t*>(o);
    }
  }

  // a previous call that failed half-way may have left staging in flight: settle it
  for (int d = 0; d < nd; ++d) {
    if (plan[d].empty()) continue;
    DeviceGuard guard(devices[d]);
    DevCtx& ctx = tl_ctx.devs[devices[d]];
    for (int i = 0; i < 2; ++i) {
      if (ctx.hout_pending[i] || ctx.hin_used[i]) {
        cudaStreamSynchronize(ctx.st[i]);
        ctx.hout_pending[i] = ctx.hin_used[i] = false;
      }
    }
  }
  const void* in_base = llr4 ? static_cast<const void*>(llr4) : static_cast<const void*>(llr);
  const bool stage_in = !host_pinned(in_base), stage_out = !host_pinned(out_packed);
  // H2D of one chunk (through the slot's pinned staging buffer when the caller's is pageable)
  auto h2d = [&](DevCtx& ctx, int slot, cudaStream_t s, void* dst, const void* src, std::size_t bytes) -> vd_status {
    if (!stage_in) {
      VD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D chunk");
      return VD_OK;
    }
    if (ctx.hin_used[slot]) VD_CUDA(cudaEventSynchronize(ctx.hin_free[slot]), "staging reuse");
    if (vd_status st = ensure_host(&ctx.hin[slot], &ctx.hin_cap[slot], bytes)) return st;
    if (!ctx.hin_free[slot]) VD_CUDA(cudaEventCreateWithFlags(&ctx.hin_free[slot], cudaEventDisableTiming), "event");
    parallel_memcpy(ctx.hin[slot], src, bytes);
    VD_CUDA(cudaMemcpyAsync(dst, ctx.hin[slot], bytes, cudaMemcpyHostToDevice, s), "H2D staged chunk");
    VD_CUDA(cudaEventRecord(ctx.hin_free[slot], s), "event");
    ctx.hin_used[slot] = true;
    return VD_OK;
  };
  auto drain = [&](DevCtx& ctx, int slot) -> vd_status {  // staged output of the slot's previous chunk -> caller
    if (!ctx.hout_pending[slot]) return VD_OK;
    VD_CUDA(cudaEventSynchronize(ctx.hout_ready[slot]), "D2H staging");
    parallel_memcpy(ctx.pend_dst[slot], ctx.hout[slot], ctx.pend_bytes[slot]);
    ctx.hout_pending[slot] = false;
    return VD_OK;
  };
  // Issue: one host thread per device (the caller's thread for the first),
  // so one device's staging copies and waits never hold up another's. Chunk
  // i of a device goes on its stream i % 2; within a stream the H2D of chunk
  // i+2 is ordered after the kernel of chunk i. Every worker uses the calling
  // thread's per-device context (each device is driven by exactly one worker).
  ThreadCtx& tctx = tl_ctx;
  auto run_device = [&](int d) -> vd_status {
    DeviceGuard guard(devices[d]);
    DevCtx& ctx = tctx.devs[devices[d]];
    for (std::size_t i = 0; i < plan[d].size(); ++i) {
      const int slot = static_cast<int>(i & 1);
      cudaStream_t s = ctx.st[slot];
      const Chunk c = plan[d][i];
      std::int64_t wb = 0, we = 0;
      if (vd_status st = vd_frame_window(cfg, n, c.f0, c.f1, &wb, &we)) return st;
      T* dl = static_cast<T*>(ctx.llr[slot]);
      if (pp) {
        const std::int64_t p0 = pp->off(wb), p1 = pp->off(we);
        if (vd_status st = h2d(ctx, slot, s, ctx.pun[slot], llr + p0, sizeof(T) * (p1 - p0))) return st;
        if (vd_status st = launch_depuncture(*pp, static_cast<const std::int8_t*>(ctx.pun[slot]), wb, we - wb,
                                             reinterpret_cast<std::int8_t*>(dl), s))
          return st;
      } else if (llr4) {
        const std::int64_t e0 = wb * code->b, e1 = we * code->b;  // element range of the chunk
        const std::int64_t by0 = e0 >> 1, by1 = (e1 + 1) >> 1;
        if (vd_status st = h2d(ctx, slot, s, ctx.pun[slot], llr4 + by0, by1 - by0)) return st;
        const cudaError_t eu = vd::launch_unpack_i4(static_cast<const std::uint8_t*>(ctx.pun[slot]),
                                                    static_cast<int>(e0 & 1), e1 - e0,
                                                    reinterpret_cast<std::int8_t*>(dl), s);
        if (eu != cudaSuccess) return cuda_fail(eu, "unpack i4 kernel");
      } else {
        if (vd_status st = h2d(ctx, slot, s, dl, llr + wb * code->b, sizeof(T) * (we - wb) * code->b)) return st;
      }
      const std::int64_t out_lo = c.f0 * cfg->f;  // multiple of 32 by construction
      const std::int64_t out_hi = std::min<std::int64_t>(c.f1 * cfg->f, n);
      vd_status st = decode_device<T>(code, cfg, n, dl, wb, c.f0, c.f1, ctx.out[slot], out_lo, nullptr, devices[d], s);
      if (st != VD_OK) return st;
      const std::int64_t words = (out_hi - out_lo + 31) / 32;
      const std::size_t obytes = sizeof(std::uint32_t) * words;
      if (!stage_out) {
        VD_CUDA(cudaMemcpyAsync(out_packed + out_lo / 32, ctx.out[slot], obytes, cudaMemcpyDeviceToHost, s),
                "D2H packed bits");
      } else {
        if (vd_status st2 = drain(ctx, slot)) return st2;
        if (vd_status st2 = ensure_host(&ctx.hout[slot], &ctx.hout_cap[slot], obytes)) return st2;
        if (!ctx.hout_ready[slot]) VD_CUDA(cudaEventCreateWithFlags(&ctx.hout_ready[slot], cudaEventDisableTiming), "event");
        VD_CUDA(cudaMemcpyAsync(ctx.hout[slot], ctx.out[slot], obytes, cudaMemcpyDeviceToHost, s), "D2H staged bits");
        VD_CUDA(cudaEventRecord(ctx.hout_ready[slot], s), "event");
        ctx.hout_pending[slot] = true;
        ctx.pend_dst[slot] = out_packed + out_lo / 32;
        ctx.pend_bytes[slot] = obytes;
      }
    }
    for (int i = 0; i < 2; ++i) {
      if (vd_status st = drain(ctx, i)) return st;
      VD_CUDA(cudaStreamSynchronize(ctx.st[i]), "decode stream");
      ctx.hin_used[i] = false;
    }
    return VD_OK;
  };
  std::vector<int> active;
  for (int d = 0; d < nd; ++d) {
    if (!plan[d].empty()) active.push_back(d);
  }
  if (active.size() <= 1) return active.empty() ? VD_OK : run_device(active[0]);
  // A device listed twice ({0, 0}) gets two chunk lists but one DevCtx: such
  // entries share a worker, which runs the lists one after the other.
  std::map<int, std::vector<int>> by_dev;
  for (int d : active) by_dev[devices[d]].push_back(d);
  std::vector<vd_status> status(by_dev.size(), VD_OK);
  std::vector<std::string> msg(by_dev.size());
  std::vector<std::thread> workers;
  auto work = [&](std::size_t w, const std::vector<int>& lst) {
    for (int d : lst) {
      status[w] = run_device(d);
      if (status[w] != VD_OK) {
        msg[w] = g_err;  // thread_local: hand the message to the caller
        return;
      }
    }
  };
  std::size_t w = 0;
  const std::vector<int>* first_list = nullptr;
  for (auto& kv : by_dev) {
    if (!first_list) {
      first_list = &kv.second;
      ++w;
      continue;
    }
    try {
      workers.emplace_back(work, w, std::cref(kv.second));
    } catch (...) {  // no thread: run it on the caller after the others
      work(w, kv.second);
    }
    ++w;
  }
  work(0, *first_list);
  for (auto& th : workers) th.join();
  for (std::size_t i = 0; i < status.size(); ++i) {
    if (status[i] != VD_OK) return fail(status[i], msg[i]);
  }
  return VD_OK;
}

}  // namespace

namespace vd {
namespace {
std::atomic<unsigned long long> g_launches{0};
}
void note_launch(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed); }

cudaError_t retain_async_pool() {
  static std::mutex mu;
  static std::map<int, bool> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  cudaMemPool_t pool;
  if (cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, dev); e != cudaSuccess) return e;
  std::uint64_t thr = ~0ull;
  if (cudaError_t e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr); e != cudaSuccess) return e;
  done[dev] = true;
  return cudaSuccess;
}

cudaError_t allow_max_smem(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
      e != cudaSuccess)
    return e;
  done.insert({kern, dev});
  return cudaSuccess;
}

int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  cache[dev] = n;
  return n;
}
}  // namespace vd

extern "C" {

const char* vd_last_error(void) { return g_err.c_str(); }
const char* vd_version(void) { return "vitdec_b200 0.2 (sm_100a)"; }
uint64_t vd_kernel_launches(void) { return vd::g_launches.load(std::memory_order_relaxed); }

vd_status vd_code_create(int32_t k, int32_t b, const uint32_t* polys, vd_code** out) {
  if (!out) return fail(VD_EINVAL, "null output handle");
  *out = nullptr;
  if (vd_status st = validate_spec(k, b, polys)) return st;
  auto c = std::make_unique<vd_code>();
  c->k = k;
  c->b = b;
  c->s = 1 << (k - 1);
  c->polys.assign(polys, polys + b);
  const int s = c->s;
  c->next.resize(2 * s);
  c->out.resize(2 * s);
  c->pred.assign(2 * s, 0);
  c->in_out.assign(2 * s, 0);
  // Tables as reference trellis.cpp:57-91.
  for (std::uint32_t st = 0; st < static_cast<std::uint32_t>(s); ++st) {
    for (std::uint32_t u = 0; u < 2; ++u) {
      const std::uint32_t reg = (u << (k - 1)) | st;
      std::uint32_t bo = 0;
      for (int i = 0; i < b; ++i) bo |= static_cast<std::uint32_t>(__builtin_popcount(polys[i] & reg) & 1) << (b - 1 - i);
      c->next[st * 2 + u] = (u << (k - 2)) | (st >> 1);
      c->out[st * 2 + u] = bo;
    }
  }
  const std::uint32_t low_mask = static_cast<std::uint32_t>(s / 2 - 1);
  for (std::uint32_t j = 0; j < static_cast<std::uint32_t>(s); ++j) {
    const std::uint32_t low = (s == 2) ? 0 : (j & low_mask);
    const std::uint32_t u = j >> (k - 2);
    for (std::uint32_t w = 0; w < 2; ++w) {
      const std::uint32_t i = low * 2 + w;
      c->pred[j * 2 + w] = i;
      c->in_out[j * 2 + w] = c->out[i * 2 + u];
    }
  }
  const std::uint32_t ones = (1u << b) - 1;
  c->complement_paired = true;
  for (int st = 0; st < s; ++st) {
    if ((c->out[st * 2] ^ c->out[st * 2 + 1]) != ones) {
      c->complement_paired = false;
      break;
    }
  }
  *out = c.release();
  return VD_OK;
}

void vd_code_destroy(vd_code* code) { delete code; }
int32_t vd_code_k(const vd_code* code) { return code ? code->k : 0; }
int32_t vd_code_b(const vd_code* code) { return code ? code->b : 0; }

vd_status vd_code_tables(const vd_code* code, uint32_t* next, uint32_t* out, uint32_t* pred, uint32_t* in_out,
                         int32_t* complement_paired) {
  if (!code) return fail(VD_EINVAL, "null code");
  const std::size_t n = code->next.size();
  if (next) std::memcpy(next, code->next.data(), n * sizeof(uint32_t));
  if (out) std::memcpy(out, code->out.data(), n * sizeof(uint32_t));
  if (pred) std::memcpy(pred, code->pred.data(), n * sizeof(uint32_t));
  if (in_out) std::memcpy(in_out, code->in_out.data(), n * sizeof(uint32_t));
  if (complement_paired) *complement_paired = code->complement_paired ? 1 : 0;
  return VD_OK;
}

int32_t vd_code_fast_path(const vd_code* code) {
  if (!code) return 0;
  vd::DecodeLaunch p;
  p.k = code->k;
  p.b = code->b;
  p.s = code->s;
  p.f = 256;
  p.v1 = p.v2 = 20;
  p.n = 1 << 20;
  p.frame_begin = 0;
  p.frame_end = p.n / p.f;
  for (int i = 0; i < code->b && i < 8; ++i) p.polys[i] = code->polys[i];
  p.complement_paired = code->complement_paired;
  return vd::fast_path_supported(p) ? 1 : 0;
}

vd_status vd_code_jit_check(const vd_code* code) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (!vd::fast_envelope_code(code->k, code->b, code->polys.data()))
    return fail(VD_EUNSUPPORTED, "code outside the fast kernel's envelope (5 <= K <= 10, B in {2, 3, 4})");
  if (!vd::jit::compile_check(code->k, code->b, code->polys.data())) return fail(VD_ECUDA, vd::jit::last_log());
  return VD_OK;
}

vd_status vd_frame_cfg_validate(const vd_frame_cfg* cfg, int32_t pattern_period) {
  return validate_cfg(cfg, pattern_period);
}

vd_status vd_frame_stats(const vd_frame_cfg* cfg, int64_t n, vd_stats* stats) {
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (!stats) return fail(VD_EINVAL, "null stats");
  // reference decoder.cpp:256-265 in closed form (O(1) instead of O(frames)):
  // interior frames are identical; only the first ceil(v1/f) and the frames
  // whose right overlap is clipped differ.
  stats->frames = num_frames(cfg, n);
  stats->stages = 0;
  stats->tracebacks = 0;
  const std::int64_t nf = stats->frames;
  auto add = [&](std::int64_t m) {
    const vd::FrameGeom g(m, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
    stats->stages += g.len();
    stats->tracebacks += g.num_sub;
  };
  const std::int64_t head = std::min<std::int64_t>(nf, (cfg->v1 + cfg->f - 1) / cfg->f + 1);
  const std::int64_t tail_start = std::max<std::int64_t>(head, nf - ((cfg->v2 + cfg->f - 1) / cfg->f + 2));
  for (std::int64_t m = 0; m < head; ++m) add(m);
  if (tail_start > head) {
    const vd::FrameGeom g(head, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
    stats->stages += g.len() * (tail_start - head);
    stats->tracebacks += g.num_sub * (tail_start - head);
  }
  for (std::int64_t m = tail_start; m < nf; ++m) add(m);
  return VD_OK;
}

vd_status vd_partition_frames(const vd_frame_cfg* cfg, int64_t n, int32_t parts, int64_t* first) {
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (parts < 1 || !first) return fail(VD_EINVAL, "bad partition request");
  const std::int64_t nf = num_frames(cfg, n);
  const std::int64_t unit = align_unit(cfg->f);
  const std::int64_t units = (nf + unit - 1) / unit;
  for (int p = 0; p <= parts; ++p) {
    first[p] = std::min<std::int64_t>(nf, (units * p / parts) * unit);
  }
  first[parts] = nf;
  return VD_OK;
}

vd_status vd_frame_window(const vd_frame_cfg* cfg, int64_t n, int64_t fb, int64_t fe, int64_t* begin, int64_t* end) {
  if (vd_status st = validate_cfg(cfg, 1)) return st;
  if (fb < 0 || fe <= fb || fe > num_frames(cfg, n)) return fail(VD_EINVAL, "frame range out of bounds");
  const vd::FrameGeom g0(fb, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
  const vd::FrameGeom g1(fe - 1, n, cfg->f, cfg->v1, cfg->v2, cfg->f0);
  *begin = g0.beg;
  *end = g1.end;
  return VD_OK;
}

vd_status vd_decode_i8_device(const vd_code* code, const vd_frame_cfg* cfg, int64_t n, const int8_t* llr,
                              int64_t llr_stage0, int64_t fb, int64_t fe, uint32_t* out, int64_t out_stage0,
                              int64_t* sigma, int32_t device, void* stream) {
  return decode_device<std::int8_t>(code, cfg, n, llr, llr_stage0, fb, fe, out, out_stage0, sigma, device, stream);
}

vd_status vd_decode_f64_device(const vd_code* code, const vd_frame_cfg* cfg, int64_t n, const double* llr,
                               int64_t llr_stage0, int64_t fb, int64_t fe, uint32_t* out, int64_t out_stage0,
                               double* sigma, int32_t device, void* stream) {
  return decode_device<double>(code, cfg, n, llr, llr_stage0, fb, fe, out, out_stage0, sigma, device, stream);
}

vd_status vd_decode_batch_i8_device(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                                    const int64_t* block_stages, const int8_t* llr, uint32_t* out, vd_stats* stats,
                                    int32_t device, void* stream) {
  return decode_batch_device<std::int8_t>(code, cfg, n_blocks, block_stages, llr, out, stats, device, stream);
}

vd_status vd_decode_batch_f64_device(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                                     const int64_t* block_stages, const double* llr, uint32_t* out, vd_stats* stats,
                                     int32_t device, void* stream) {
  return decode_batch_device<double>(code, cfg, n_blocks, block_stages, llr, out, stats, device, stream);
}

vd_status vd_decode_batch_i8(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                             const int64_t* block_stages, const int8_t* llr, uint32_t* out, vd_stats* stats,
                             const vd_exec* exec) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (n_blocks < 1 || !block_stages) return fail(VD_EINVAL, "batch needs at least one block");
  std::int64_t n = 0;
  for (std::int32_t j = 0; j < n_blocks; ++j) n += block_stages[j] > 0 ? block_stages[j] : 0;
  int dev = 0;
  if (vd_status st = resolve_device(exec && exec->num_devices > 0 && exec->devices ? exec->devices[0] : -1, &dev))
    return st;
  DeviceGuard guard(dev);
  DevCtx& ctx = tl_ctx.devs[dev];
  if (!ctx.st[0]) VD_CUDA(cudaStreamCreateWithFlags(&ctx.st[0], cudaStreamNonBlocking), "cudaStreamCreate");
  const std::size_t words = static_cast<std::size_t>((n + 31) / 32);
  if (vd_status st = ensure(&ctx.llr[0], &ctx.llr_cap[0], static_cast<std::size_t>(n) * code->b)) return st;
  if (vd_status st = ensure(reinterpret_cast<void**>(&ctx.out[0]), &ctx.out_cap[0], words * 4)) return st;
  cudaStream_t s = ctx.st[0];
  VD_CUDA(cudaMemcpyAsync(ctx.llr[0], llr, static_cast<std::size_t>(n) * code->b, cudaMemcpyHostToDevice, s), "H2D");
  if (vd_status st = decode_batch_device<std::int8_t>(code, cfg, n_blocks, block_stages,
                                                      static_cast<const std::int8_t*>(ctx.llr[0]), ctx.out[0], stats,
                                                      dev, s))
    return st;
  VD_CUDA(cudaMemcpyAsync(out, ctx.out[0], words * 4, cudaMemcpyDeviceToHost, s), "D2H");
  VD_CUDA(cudaStreamSynchronize(s), "batched decode");
  return VD_OK;
}

vd_status vd_decode_i8(const vd_code* code, const vd_frame_cfg* cfg, const int8_t* llr, int64_t n, uint32_t* out,
                       vd_stats* stats, const vd_exec* exec) {
  return decode_host<std::int8_t>(code, cfg, llr, n, out, stats, exec);
}

vd_status vd_decode_f64(const vd_code* code, const vd_frame_cfg* cfg, const double* llr, int64_t n, uint32_t* out,
                        vd_stats* stats, const vd_exec* exec) {
  return decode_host<double>(code, cfg, llr, n, out, stats, exec);
}

vd_status vd_puncture_validate(const vd_puncture* pattern) {
  PunctPlan pp;
  return make_punct(pattern, &pp);
}

vd_status vd_depuncture_stages(const vd_puncture* pattern, int64_t n_punctured, int64_t* n_stages) {
  PunctPlan pp;
  if (vd_status st = make_punct(pattern, &pp)) return st;
  if (!n_stages) return fail(VD_EINVAL, "null buffer");
  return punct_stages(pp, n_punctured, n_stages);
}

vd_status vd_depuncture_f64(const vd_puncture* pattern, const double* punctured, int64_t n_punctured,
                            double* llr_out) {
  PunctPlan pp;
  if (vd_status st = make_punct(pattern, &pp)) return st;
  std::int64_t n = 0;
  if (vd_status st = punct_stages(pp, n_punctured, &n)) return st;
  if (n == 0) return VD_OK;
  if (!punctured || !llr_out) return fail(VD_EINVAL, "null buffer");
  int dev = 0;
  if (vd_status st = resolve_device(-1, &dev)) return st;
  DeviceGuard guard(dev);
  DevCtx& ctx = tl_ctx.devs[dev];
  if (!ctx.st[0]) VD_CUDA(cudaStreamCreateWithFlags(&ctx.st[0], cudaStreamNonBlocking), "cudaStreamCreate");
  cudaStream_t s = ctx.st[0];
  VD_CUDA(vd::retain_async_pool(), "memory pool");
  double* din = nullptr;
  double* dout = nullptr;
  const std::size_t in_bytes = sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(n_punctured, 1));
  const std::size_t out_bytes = sizeof(double) * static_cast<std::size_t>(n) * pp.b;
  VD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&din), in_bytes, s), "cudaMallocAsync(depuncture in)");
  VD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), out_bytes, s), "cudaMallocAsync(depuncture out)");
  cudaError_t e = cudaMemcpyAsync(din, punctured, sizeof(double) * n_punctured, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = vd::launch_depuncture_f64(din, n, pp.b, pp.period, pp.kept, pp.rank.data(), dout, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(llr_out, dout, out_bytes, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(din, s);
  cudaFreeAsync(dout, s);
  const cudaError_t es = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "depuncture");
  if (es != cudaSuccess) return cuda_fail(es, "depuncture");
  return VD_OK;
}

vd_status vd_depuncture_i8_device(const vd_puncture* pattern, const int8_t* punctured_dev, int64_t n_punctured,
                                  int8_t* llr_dev, int32_t device, void* stream) {
  PunctPlan pp;
  if (vd_status st = make_punct(pattern, &pp)) return st;
  std::int64_t n = 0;
  if (vd_status st = punct_stages(pp, n_punctured, &n)) return st;
  if (n == 0) return VD_OK;
  if (!punctured_dev || !llr_dev) return fail(VD_EINVAL, "null buffer");
  if (reinterpret_cast<std::uintptr_t>(llr_dev) & 3u) return fail(VD_EINVAL, "llr_dev must be 4-byte aligned");
  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  return launch_depuncture(pp, punctured_dev, 0, n, llr_dev, static_cast<cudaStream_t>(stream));
}

// framed_decode(depuncture(stream, pattern), trellis, cfg): the composition
// the reference's BER harness and CLI run (berlab.cpp:79-84, vitdec_cli.cpp:172-176).
static vd_status punct_decode_prep(const vd_code* code, const vd_frame_cfg* cfg, const vd_puncture* pattern,
                                   int64_t n_punctured, PunctPlan* pp, std::int64_t* n) {
  if (!code) return fail(VD_EINVAL, "null code");
  if (vd_status st = make_punct(pattern, pp)) return st;
  if (vd_status st = punct_stages(*pp, n_punctured, n)) return st;
  if (*n < 1) return fail(VD_EINVAL, "empty llr block");
  if (pp->b != code->b) return fail(VD_EINVAL, "llr row count must equal B");  // check_block, decoder.cpp:92-97
  return validate_cfg(cfg, 1);
}

vd_status vd_decode_punctured_i8(const vd_code* code, const vd_frame_cfg* cfg, const vd_puncture* pattern,
                                 const int8_t* punctured, int64_t n_punctured, uint32_t* out_packed, vd_stats* stats,
                                 const vd_exec* exec) {
  PunctPlan pp;
  std::int64_t n = 0;
  if (vd_status st = punct_decode_prep(code, cfg, pattern, n_punctured, &pp, &n)) return st;
  return decode_host<std::int8_t>(code, cfg, punctured, n, out_packed, stats, exec, &pp);
}

vd_status vd_decode_punctured_i8_device(const vd_code* code, const vd_frame_cfg* cfg, const vd_puncture* pattern,
                                        const int8_t* punctured_dev, int64_t n_punctured, int8_t* llr_scratch_dev,
                                        uint32_t* out_dev, vd_stats* stats, int32_t device, void* stream) {
  PunctPlan pp;
  std::int64_t n = 0;
  if (vd_status st = punct_decode_prep(code, cfg, pattern, n_punctured, &pp, &n)) return st;
  if (stats) {
    if (vd_status st = vd_frame_stats(cfg, n, stats)) return st;
  }
  if (!punctured_dev || !llr_scratch_dev || !out_dev) return fail(VD_EINVAL, "null buffer");
  if (reinterpret_cast<std::uintptr_t>(llr_scratch_dev) & 3u) return fail(VD_EINVAL, "llr_scratch_dev must be 4-byte aligned");
  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const std::int64_t nf = num_frames(cfg, n);
  // Fused depuncture (vd_fast_dev.cuh Punct; the default, VITDEC_PUNCT_FUSED=0
  // turns it off): the fast kernel stages the punctured stream straight into
  // its shared-memory LLR ring; the few edge frames it does not take are
  // decoded from dense copies of their windows on the side stream. Measured
  // against the separate HBM-streaming depuncture pass + decode on one B200
  // (2^30 stages, f=240/24/24): 1.05x (r2/3), 1.04x (r3/4)
  // (profiles/r02_puncture_bench.jsonl, profiles/r02_ab_notes.md).
  const int pid = punct_pattern_id(pp);
  const char* env_fused = std::getenv("VITDEC_PUNCT_FUSED");
  const bool want_fused = pid != 0 && !(env_fused && std::atoi(env_fused) == 0) &&
                          (reinterpret_cast<std::uintptr_t>(punctured_dev) & 3u) == 0 && cfg->f0 == 0;
  if (want_fused && check_gpu_envelope(code) == VD_OK) {
    vd::DecodeLaunch p;
    p.k = code->k;
    p.b = code->b;
    p.s = code->s;
    p.f = cfg->f;
    p.v1 = cfg->v1;
    p.v2 = cfg->v2;
    p.f0 = cfg->f0;
    p.start = cfg->start;
    p.seed = cfg->seed;
    p.n = n;
    p.frame_begin = 0;
    p.frame_end = nf;
    p.llr = punctured_dev;
    p.llr_stage0 = 0;
    p.out = out_dev;
    for (int i = 0; i < code->b && i < 8; ++i) p.polys[i] = code->polys[i];
    p.complement_paired = code->complement_paired;
    std::int64_t mi0 = 0, mi1 = 0;
    if (vd::launch_fast_punct_i8(p, pid, nullptr, nullptr, &mi0, &mi1) && mi1 > mi0) {
      const std::uint32_t* in_out = nullptr;
      if (vd_status st = device_table(code, dev, &in_out)) return st;
      p.in_out = in_out;
      // Every output word is zeroed first (all kernels OR their bits in;
      // edge and interior frames share at most the two boundary words), then
      // the edge frames — each decoded from a dense depunctured copy of its
      // window — run on the side stream beside the fused kernel.
      VD_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(std::uint32_t) * static_cast<std::size_t>((n + 31) / 32), s),
              "zero output");
      const bool edges = mi0 > 0 || mi1 < nf;
      cudaStream_t side = nullptr;
      if (edges) VD_CUDA(vd::side_fork(s, &side), "side stream");
      auto decode_edge = [&](std::int64_t llr_stage0, std::int64_t fb, std::int64_t fe, std::int64_t out_stage0) {
        vd::DecodeLaunch e = p;
        e.llr = llr_scratch_dev;
        e.llr_stage0 = llr_stage0;
        e.frame_begin = fb;
        e.frame_end = fe;
        e.out = out_dev + out_stage0 / 32;
        e.out_stage0 = out_stage0;
        return vd::fast_path_supported(e) ? vd::launch_fast_i8(e, side) : vd::launch_generic_i8(e, side);
      };
      if (mi0 > 0) {
        const std::int64_t t1 = std::min<std::int64_t>(mi0 * cfg->f + cfg->v2 + vd::kPfSlackStages, n);
        if (vd_status st = launch_depuncture(pp, punctured_dev, 0, t1, llr_scratch_dev, side)) return st;
        VD_CUDA(decode_edge(0, 0, mi0, 0), "edge frames");
      }
      if (mi1 < nf) {
        const std::int64_t t0 = mi1 * cfg->f - cfg->v1;  // a period multiple: f and v1 are
        if (vd_status st = launch_depuncture(pp, punctured_dev + pp.off(t0), t0, n - t0, llr_scratch_dev, side))
          return st;
        VD_CUDA(decode_edge(t0, mi1, nf, (mi1 * cfg->f) / 32 * 32), "edge frames");
      }
      cudaError_t e = cudaSuccess;
      if (!vd::launch_fast_punct_i8(p, pid, s, &e, &mi0, &mi1)) return fail(VD_ECUDA, "fused depuncture plan changed");
      if (e != cudaSuccess) return cuda_fail(e, "fused depuncture decode");
      if (edges) VD_CUDA(vd::side_join(s), "side stream");
      return VD_OK;
    }
  }
  if (vd_status st = launch_depuncture(pp, punctured_dev, 0, n, llr_scratch_dev, s)) return st;
  return decode_device<std::int8_t>(code, cfg, n, llr_scratch_dev, 0, 0, nf, out_dev, 0, nullptr, dev, stream);
}

vd_status vd_decode_i4(const vd_code* code, const vd_frame_cfg* cfg, const uint8_t* llr4, int64_t n, uint32_t* out,
                       vd_stats* stats, const vd_exec* exec) {
  if (!llr4) return fail(VD_EINVAL, "null buffer");
  return decode_host<std::int8_t>(code, cfg, reinterpret_cast<const std::int8_t*>(llr4), n, out, stats, exec, nullptr,
                                  llr4);
}

vd_status vd_unpack_i4_device(const uint8_t* llr4_dev, int64_t count, int8_t* llr_dev, int32_t device, void* stream) {
  if (count < 0) return fail(VD_EINVAL, "negative count");
  if (count == 0) return VD_OK;
  if (!llr4_dev || !llr_dev) return fail(VD_EINVAL, "null buffer");
  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  const cudaError_t e = vd::launch_unpack_i4(llr4_dev, 0, count, llr_dev, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorMisalignedAddress) return fail(VD_EINVAL, "llr4_dev must be 4-byte and llr_dev 8-byte aligned");
  if (e != cudaSuccess) return cuda_fail(e, "unpack i4 kernel");
  return VD_OK;
}

vd_status vd_serial_decode_f64(const vd_code* code, const double* llr, int64_t n, uint32_t* out, vd_stats* stats,
                               int32_t device) {
  if (n < 1) return fail(VD_EINVAL, "empty llr block");
  if (n > 0x7fffffffLL) return fail(VD_EUNSUPPORTED, "serial decode limited to 2^31-1 stages");
  vd_frame_cfg cfg{};
  cfg.f = static_cast<int32_t>(n);
  vd_exec ex{};
  int32_t dev = device;
  if (device >= 0) {
    ex.num_devices = 1;
    ex.devices = &dev;
  }
  ex.chunk_stages = n;
  return decode_host<double>(code, &cfg, llr, n, out, stats, &ex);
}

vd_status vd_synth_llr_i8_device(const vd_code* code, int64_t n, double sigma, double scale, uint64_t seed,
                                 int8_t* llr, uint32_t* bits, int32_t device, void* stream) {
  return vd_synth_llr_i8_range_device(code, 0, n, sigma, scale, seed, llr, bits, device, stream);
}

vd_status vd_synth_llr_i8_range_device(const vd_code* code, int64_t t_begin, int64_t n, double sigma, double scale,
                                       uint64_t seed, int8_t* llr, uint32_t* bits, int32_t device, void* stream) {
  if (!code || (!llr && !bits) || n < 1 || t_begin < 0) return fail(VD_EINVAL, "bad synth arguments");
  if (bits && (t_begin & 31)) return fail(VD_EINVAL, "message bits need t_begin % 32 == 0");
  if (code->b > 4) return fail(VD_EUNSUPPORTED, "synthetic generator supports B <= 4");
  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  const cudaError_t e = vd::launch_synth_i8(code->k, code->b, code->polys.data(), t_begin, n, sigma, scale, seed, llr, bits,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "synth kernel");
  return VD_OK;
}

vd_status vd_count_bit_errors_device(const uint32_t* a, const uint32_t* b, int64_t n_bits, unsigned long long* count,
                                     int32_t device, void* stream) {
  if (!a || !b || !count) return fail(VD_EINVAL, "null buffer");
  int dev = 0;
  if (vd_status st = resolve_device(device, &dev)) return st;
  DeviceGuard guard(dev);
  const cudaError_t e = vd::launch_count_bit_errors(a, b, n_bits, count, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "bit-error count kernel");
  return VD_OK;
}

}  // extern "C"
