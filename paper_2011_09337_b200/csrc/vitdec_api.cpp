// The reference C++ decoder API (include/vitdec/{trellis,decoder}.hpp)
// implemented over the vitdec_b200 C-ABI. This file replaces the reference's
// trellis.cpp and decoder.cpp in a link: the decode entry points call the
// GPU, everything else keeps the reference's semantics and exception
// messages.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <sys/mman.h>

#include "vitdec/decoder.hpp"
#include "vitdec/trellis.hpp"
#include "vitdec_b200.h"
#include "vd_host_convert.h"

namespace vitdec {
namespace {

#ifdef MADV_POPULATE_WRITE
constexpr int kMadvPopulateWrite = MADV_POPULATE_WRITE;
#else
constexpr int kMadvPopulateWrite = 23;  // Linux >= 5.14
#endif

[[noreturn]] void raise(vd_status st) {
  const std::string msg = vd_last_error();
  if (st == VD_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("vitdec_b200: " + msg);
}

void check(vd_status st) {
  if (st != VD_OK) raise(st);
}

vd_frame_cfg to_c(const FrameConfig& cfg) {
  vd_frame_cfg c{};
  c.f = cfg.f;
  c.v1 = cfg.v1;
  c.v2 = cfg.v2;
  c.f0 = cfg.f0;
  c.start = cfg.start == TracebackStart::kRandom ? VD_TB_RANDOM : VD_TB_STORED_MAX;
  c.seed = cfg.seed;
  return c;
}

DecodeStats from_c(const vd_stats& s) {
  DecodeStats o;
  o.frames = s.frames;
  o.stages = s.stages;
  o.tracebacks = s.tracebacks;
  return o;
}

// reference decoder.cpp:92-97
void check_block(const LlrBlock& llr, const Trellis& trellis) {
  if (llr.cols() < 1) throw std::invalid_argument("empty llr block");
  if (llr.rows() != trellis.outputs_per_bit()) throw std::invalid_argument("llr row count must equal B");
}

// VITDEC_GPUS=N shards the drop-in decode over devices 0 .. N-1; unset (or
// <= 0) decodes on the calling thread's current device (vd_exec num_devices 0).
int env_gpus() {
  const char* v = std::getenv("VITDEC_GPUS");
  if (!v || !*v) return 0;
  const int g = std::atoi(v);
  return g > 0 ? g : 0;
}

// Runs fn(lo, hi) over [0, n) on `workers` host threads (the reference's
// `workers` argument, parallel.hpp:11-29 semantics: contiguous chunks, joined
// before return); small ranges stay on the calling thread.
template <typename Fn>
void host_parallel(std::int64_t n, int workers, Fn&& fn) {
  const std::int64_t w = std::max<std::int64_t>(1, std::min<std::int64_t>(workers, n / (1 << 20) + 1));
  if (w <= 1) {
    fn(std::int64_t{0}, n);
    return;
  }
  const std::int64_t chunk = (n + w - 1) / w;
  std::vector<std::thread> th;
  for (std::int64_t i = 0; i < w; ++i) {
    const std::int64_t lo = i * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : th) t.join();
}

// Per-thread pinned host buffers for the converted int8 block and the packed
// result of the drop-in framed_decode: H2D / D2H go straight from / to them
// (no staging copy) and repeated calls reuse them (no fresh pages per call).
// Grown on demand; plain heap memory when pinned memory is unavailable.
constexpr std::size_t kMaxPinned = std::size_t{512} << 20;
struct HostScratch {
  void* p[2] = {nullptr, nullptr};
  std::size_t cap[2] = {0, 0};
  bool pinned[2] = {false, false};
  ~HostScratch() {
    for (int i = 0; i < 2; ++i) release(i);
  }
  void release(int i) {
    if (!p[i]) return;
    if (pinned[i]) {
      cudaFreeHost(p[i]);
    } else {
      std::free(p[i]);
    }
    p[i] = nullptr;
    cap[i] = 0;
  }
  void* get(int i, std::size_t bytes) {
    if (cap[i] >= bytes) return p[i];
    release(i);
    const std::size_t want = std::max<std::size_t>(bytes, cap[i] + cap[i] / 2);
    // (pinned up to kMaxPinned per buffer: larger blocks use pageable memory,
    // which the library stages through its own pinned chunks)
    pinned[i] = want <= kMaxPinned && cudaMallocHost(&p[i], want) == cudaSuccess;
    if (!pinned[i]) {
      cudaGetLastError();
      p[i] = std::malloc(want);
      if (!p[i]) throw std::bad_alloc();
    }
    cap[i] = want;
    return p[i];
  }
};
thread_local HostScratch t_scratch;

// True when every value is an integer in [-127, 127]: the block is then
// decoded by the int8 fixed-point kernels, exactly (integer sums are exact in
// both the reference's double arithmetic and the kernel's int32 arithmetic).
bool int8_exact(const LlrBlock& llr, std::int8_t* out, int workers) {
  const double* d = llr.data();
  std::atomic<bool> ok{true};
  host_parallel(llr.size(), workers, [&](std::int64_t lo, std::int64_t hi) {
    if (host::int8_range(d, out, lo, hi)) ok.store(false, std::memory_order_relaxed);
  });
  return ok.load();
}

// A BitVec of n bytes whose pages are already faulted in. A fresh multi-MiB
// vector is an mmap, and first-touch faults in the single-threaded zero-fill
// of std::vector's constructor cost more than the decode (2^26 bits: 23 ms);
// its 2 MiB-aligned interior is advised to huge pages, then `workers` threads
// fault their own ranges in first (MADV_POPULATE_WRITE).
BitVec resident_bits(Eigen::Index n, int workers) {
  BitVec bits;
  bits.reserve(static_cast<std::size_t>(n));
  constexpr std::uintptr_t kPage = 4096;
  if (n >= (std::int64_t{4} << 20)) {
    const auto base = reinterpret_cast<std::uintptr_t>(bits.data());
    {  // 2 MiB pages where transparent huge pages are on "madvise": 512x fewer
       // faults (reference-API e2e at 2^26 bits 2.2 -> 2.6 Gbps; advisory)
      constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20;
      const std::uintptr_t a = (base + kHuge - 1) & ~(kHuge - 1), b = (base + n) & ~(kHuge - 1);
      if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
    }
    host_parallel(n, workers, [&](std::int64_t lo, std::int64_t hi) {
      const std::uintptr_t a = (base + lo + kPage - 1) & ~(kPage - 1), b = (base + hi) & ~(kPage - 1);
      if (b > a) madvise(reinterpret_cast<void*>(a), b - a, kMadvPopulateWrite);  // (advisory: failure is harmless)
    });
  }
  bits.resize(static_cast<std::size_t>(n));
  return bits;
}

// One byte per bit from the packed words, 8 bytes per table lookup.
void unpack_into(BitVec& bits, const std::uint32_t* packed, Eigen::Index n, int workers = 1) {
  static const auto lut = [] {
    std::array<std::uint64_t, 256> t{};
    for (int v = 0; v < 256; ++v)
      for (int j = 0; j < 8; ++j) t[v] |= static_cast<std::uint64_t>((v >> j) & 1) << (8 * j);
    return t;
  }();
  std::uint8_t* out = bits.data();
  const std::int64_t nbytes = n / 8;  // whole packed bytes
  const auto* pb = reinterpret_cast<const std::uint8_t*>(packed);  // (little-endian: bit i is bit i % 8 of byte i / 8)
  host_parallel(nbytes, workers, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t j = lo; j < hi; ++j) std::memcpy(out + 8 * j, &lut[pb[j]], 8);
  });
  for (std::int64_t i = 8 * nbytes; i < n; ++i) out[i] = static_cast<std::uint8_t>((packed[i >> 5] >> (i & 31)) & 1u);
}

BitVec unpack(const std::uint32_t* packed, Eigen::Index n) {
  BitVec bits(static_cast<std::size_t>(n));
  unpack_into(bits, packed, n);
  return bits;
}

// Runs fn on its own thread from construction; joined by wait() or the
// destructor (also on an exception unwinding the caller).
class Background {
 public:
  template <typename Fn>
  explicit Background(Fn&& fn) : th_(std::forward<Fn>(fn)) {}
  ~Background() { wait(); }
  void wait() {
    if (th_.joinable()) th_.join();
  }

 private:
  std::thread th_;
};

}  // namespace

// ---- trellis.hpp ---------------------------------------------------------

CodeSpec CodeSpec::from_octal(int k, const std::string& octal_csv) {
  CodeSpec spec;
  spec.k = k;
  std::stringstream ss(octal_csv);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) continue;
    std::size_t used = 0;
    const unsigned long v = std::stoul(tok, &used, 8);
    if (used != tok.size()) throw std::invalid_argument("bad octal polynomial: " + tok);
    spec.polys.push_back(static_cast<std::uint32_t>(v));
  }
  spec.b = static_cast<int>(spec.polys.size());
  return spec;
}

std::string CodeSpec::polys_octal() const {
  std::ostringstream os;
  for (std::size_t i = 0; i < polys.size(); ++i) os << (i ? "," : "") << std::oct << polys[i] << std::dec;
  return os.str();
}

Trellis::Trellis(const CodeSpec& spec) : spec_(spec) {
  // reference trellis.cpp:38-53 ordering: a polys/B count mismatch is
  // reported before the C-ABI sees the (possibly short) array.
  if (spec.k >= 2 && spec.b >= 2 && static_cast<int>(spec.polys.size()) != spec.b) {
    throw std::invalid_argument("polynomial count must equal B");
  }
  vd_code* raw = nullptr;
  std::vector<std::uint32_t> polys = spec.polys;
  polys.resize(static_cast<std::size_t>(spec.b > 0 ? spec.b : 0), 0);
  check(vd_code_create(spec.k, spec.b, polys.data(), &raw));
  code_.reset(raw, vd_code_destroy);
  num_states_ = 1 << (spec.k - 1);
  const std::size_t n = static_cast<std::size_t>(num_states_) * 2;
  next_.resize(n);
  out_.resize(n);
  pred_.resize(n);
  in_out_.resize(n);
  std::int32_t cp = 0;
  check(vd_code_tables(raw, next_.data(), out_.data(), pred_.data(), in_out_.data(), &cp));
  complement_paired_ = cp != 0;
}

Trellis build_trellis(const CodeSpec& spec) { return Trellis(spec); }

// ---- decoder.hpp: configuration and per-stage helpers ----------------------

void FrameConfig::validate(int pattern_period) const {
  const vd_frame_cfg c = to_c(*this);
  check(vd_frame_cfg_validate(&c, pattern_period));
}

// reference decoder.cpp:22-30 (sum in b order from 0.0)
double branch_metric(std::uint32_t bo, const Eigen::Ref<const Eigen::ArrayXd>& llr_t) {
  const int b = static_cast<int>(llr_t.size());
  double m = 0.0;
  for (int i = 0; i < b; ++i) m += ((bo >> (b - 1 - i)) & 1u) ? -llr_t[i] : llr_t[i];
  return m;
}

// reference decoder.cpp:32-39
Eigen::ArrayXd stage_metrics(const Eigen::Ref<const Eigen::ArrayXd>& llr_t) {
  const int b = static_cast<int>(llr_t.size());
  Eigen::ArrayXd half(Eigen::Index{1} << (b - 1));
  for (Eigen::Index bo = 0; bo < half.size(); ++bo) half[bo] = branch_metric(static_cast<std::uint32_t>(bo), llr_t);
  return half;
}

// reference decoder.cpp:41-51
void fill_stage_table(const Eigen::Ref<const Eigen::ArrayXd>& llr_t, double* table) {
  const int b = static_cast<int>(llr_t.size());
  const std::uint32_t all = (1u << b) - 1;
  for (std::uint32_t bo = 0; bo < (1u << (b - 1)); ++bo) table[bo] = branch_metric(bo, llr_t);
  for (std::uint32_t bo = 1u << (b - 1); bo <= all; ++bo) table[bo] = -table[bo ^ all];
}

// reference decoder.cpp:53-76 (strict '>', ties to the second predecessor)
void acs_stage(const Eigen::ArrayXd& sigma_prev, const double* stage_table, const Trellis& trellis,
               Eigen::ArrayXd& sigma_cur, std::uint16_t* pi_col) {
  const int s = trellis.num_states();
  const std::uint32_t low = static_cast<std::uint32_t>(s / 2 - 1);
  const std::uint32_t* io = trellis.incoming_output_data();
  for (int j = 0; j < s; ++j) {
    const std::uint32_t i1 = (static_cast<std::uint32_t>(j) & low) << 1;
    const double a = sigma_prev[i1] + stage_table[io[2 * j]];
    const double c = sigma_prev[i1 | 1] + stage_table[io[2 * j + 1]];
    const bool second = !(a > c);
    sigma_cur[j] = second ? c : a;
    pi_col[j] = static_cast<std::uint16_t>(second ? (i1 | 1) : i1);
  }
}

// reference decoder.cpp:131-163 (depuncture): validation and the stage count
// through the C-ABI (vd_depuncture_stages, same messages), the gather itself
// on the device (vd_depuncture_f64); LlrBlock is column-major B x N, i.e. the
// stage-major stream the kernel writes.
LlrBlock depuncture(const Eigen::Ref<const Eigen::ArrayXd>& punctured, const PuncturePattern& p) {
  if (static_cast<int>(p.mask.size()) != p.b * p.period) throw std::invalid_argument("puncture mask shape mismatch");
  const vd_puncture pc{p.b, p.period, p.mask.data()};
  std::int64_t stages = 0;
  check(vd_depuncture_stages(&pc, punctured.size(), &stages));
  LlrBlock block = LlrBlock::Zero(p.b, stages);
  if (stages == 0) return block;
  const Eigen::ArrayXd in = punctured;  // contiguous copy (Ref may be strided)
  check(vd_depuncture_f64(&pc, in.data(), in.size(), block.data()));
  return block;
}

// ---- decoder.hpp: GPU decode entry points ---------------------------------

DecodeOutput framed_decode(const LlrBlock& llr, const Trellis& trellis, const FrameConfig& cfg, int workers) {
  check_block(llr, trellis);
  cfg.validate();
  const vd_frame_cfg c = to_c(cfg);
  const Eigen::Index n = llr.cols();
  auto* packed = static_cast<std::uint32_t*>(t_scratch.get(1, sizeof(std::uint32_t) * static_cast<std::size_t>((n + 31) / 32)));
  vd_stats st{};
  vd_exec ex{};
  ex.num_devices = env_gpus();
  auto* q = static_cast<std::int8_t*>(t_scratch.get(0, static_cast<std::size_t>(llr.size())));
  // the returned bits' pages are faulted in beside the conversion and decode
  DecodeOutput out;
  Background prep([&out, n, workers] { out.bits = resident_bits(n, std::max(1, workers / 4)); });
  // `workers` host threads prepare the block / unpack the bits (the GPU does the decode)
  const auto t0 = std::chrono::steady_clock::now();
  const bool i8 = int8_exact(llr, q, workers);
  const auto t1 = std::chrono::steady_clock::now();
  if (i8) {
    check(vd_decode_i8(trellis.native(), &c, q, n, packed, &st, &ex));
  } else {
    check(vd_decode_f64(trellis.native(), &c, llr.data(), n, packed, &st, &ex));
  }
  const auto t2 = std::chrono::steady_clock::now();
  prep.wait();
  const auto t3 = std::chrono::steady_clock::now();
  unpack_into(out.bits, packed, n, workers);
  const auto t4 = std::chrono::steady_clock::now();
  if (std::getenv("VITDEC_DROPIN_TIMING")) {  // (phase breakdown on stderr)
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "dropin: convert %.2f decode %.2f wait-pages %.2f unpack %.2f ms\n", ms(t0, t1), ms(t1, t2),
                 ms(t2, t3), ms(t3, t4));
  }
  out.stats = from_c(st);
  return out;
}

DecodeOutput serial_decode(const LlrBlock& llr, const Trellis& trellis) {
  check_block(llr, trellis);
  const Eigen::Index n = llr.cols();
  std::vector<std::uint32_t> packed(static_cast<std::size_t>((n + 31) / 32));
  vd_stats st{};
  std::vector<std::int8_t> q(static_cast<std::size_t>(llr.size()));
  if (n <= 0x7fffffff && int8_exact(llr, q.data(), 1)) {
    // One frame covering the block with no overlap == serial_decode
    // (reference acceptance.cpp:57-81 equivalence).
    vd_frame_cfg c{};
    c.f = static_cast<std::int32_t>(n);
    vd_exec ex{};
    ex.chunk_stages = n;
    check(vd_decode_i8(trellis.native(), &c, q.data(), n, packed.data(), &st, &ex));
  } else {
    check(vd_serial_decode_f64(trellis.native(), llr.data(), n, packed.data(), &st, -1));
  }
  DecodeOutput out;
  out.bits = unpack(packed.data(), n);
  out.stats = from_c(st);
  return out;
}

DecodeStats framed_decode(const std::int8_t* llr, std::int64_t n_stages, const Trellis& trellis,
                          const FrameConfig& cfg, std::uint32_t* packed_out, const ExecOptions& exec) {
  cfg.validate();
  const vd_frame_cfg c = to_c(cfg);
  vd_stats st{};
  vd_exec ex{};
  ex.num_devices = exec.gpus > 0 ? exec.gpus : 0;
  ex.chunk_stages = exec.chunk_stages;
  check(vd_decode_i8(trellis.native(), &c, llr, n_stages, packed_out, &st, &ex));
  return from_c(st);
}

DecodeStats framed_decode_punctured(const std::int8_t* punctured, std::int64_t n_punctured,
                                    const PuncturePattern& pattern, const Trellis& trellis, const FrameConfig& cfg,
                                    std::uint32_t* packed_out, const ExecOptions& exec) {
  cfg.validate();
  const vd_frame_cfg c = to_c(cfg);
  const vd_puncture pc{pattern.b, pattern.period, pattern.mask.data()};
  if (static_cast<int>(pattern.mask.size()) != pattern.b * pattern.period) {
    throw std::invalid_argument("puncture mask shape mismatch");
  }
  vd_stats st{};
  vd_exec ex{};
  ex.num_devices = exec.gpus > 0 ? exec.gpus : 0;
  ex.chunk_stages = exec.chunk_stages;
  check(vd_decode_punctured_i8(trellis.native(), &c, &pc, punctured, n_punctured, packed_out, &st, &ex));
  return from_c(st);
}

}  // namespace vitdec
