// C wrapper around the REFERENCE implementation (test infrastructure only).
//
// This file is compiled together with the reference's own, unmodified
// sources (/root/reference/proj/src/{trellis,codec,channel,decoder,berlab}.cpp,
// read in place, never copied) into oracle/_ref/libvitdec_ref.so by
// oracle/Makefile. It exposes the reference's hot path and its data chain to
// ctypes so tests can (a) pin the C restatement in oracle/vd_oracle.c against
// the real reference, (b) generate golden fixtures, and (c) serve as the
// `cpu_baseline.kind == "reference"` arm of bench.py. Nothing in the product
// path links or loads this library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "vitdec/berlab.hpp"
#include "vitdec/channel.hpp"
#include "vitdec/codec.hpp"
#include "vitdec/decoder.hpp"
#include "vitdec/trellis.hpp"

namespace {

thread_local std::string g_err;

vitdec::CodeSpec make_spec(int k, int b, const std::uint32_t* polys) {
  vitdec::CodeSpec spec;
  spec.k = k;
  spec.b = b;
  spec.polys.assign(polys, polys + b);
  return spec;
}

vitdec::FrameConfig make_cfg(int f, int v1, int v2, int f0, int start, std::uint64_t seed) {
  vitdec::FrameConfig cfg;
  cfg.f = f;
  cfg.v1 = v1;
  cfg.v2 = v2;
  cfg.f0 = f0;
  cfg.start = start ? vitdec::TracebackStart::kRandom : vitdec::TracebackStart::kStoredMax;
  cfg.seed = seed;
  return cfg;
}

void put_out(const vitdec::DecodeOutput& out, std::uint8_t* bits, std::int64_t* stats) {
  std::memcpy(bits, out.bits.data(), out.bits.size());
  if (stats) {
    stats[0] = out.stats.frames;
    stats[1] = out.stats.stages;
    stats[2] = out.stats.tracebacks;
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* vdref_last_error(void) { return g_err.c_str(); }

std::uint64_t vdref_mix_seed(std::uint64_t seed, std::uint64_t salt) { return vitdec::mix_seed(seed, salt); }

double vdref_sigma_from_ebn0(double ebn0_db, double rate) { return vitdec::sigma_from_ebn0(ebn0_db, rate); }

/// Trellis tables, each [S*2]. Returns complement_paired in *cp.
int vdref_trellis(int k, int b, const std::uint32_t* polys, std::uint32_t* next, std::uint32_t* out,
                  std::uint32_t* pred, std::uint32_t* in_out, int* cp) {
  return guarded([&] {
    const vitdec::Trellis t = vitdec::build_trellis(make_spec(k, b, polys));
    const int s = t.num_states();
    for (int i = 0; i < s; ++i) {
      for (int u = 0; u < 2; ++u) {
        next[i * 2 + u] = t.next_state(i, u);
        out[i * 2 + u] = t.branch_output(i, u);
      }
      pred[i * 2] = t.predecessors(i).first;
      pred[i * 2 + 1] = t.predecessors(i).second;
      in_out[i * 2] = t.incoming_output(i, 0);
      in_out[i * 2 + 1] = t.incoming_output(i, 1);
    }
    *cp = t.complement_paired() ? 1 : 0;
  });
}

/// Reference framed_decode on a B x n stage-major double stream.
int vdref_framed_decode_f64(int k, int b, const std::uint32_t* polys, const double* llr, std::int64_t n, int f,
                            int v1, int v2, int f0, int start, std::uint64_t seed, int workers,
                            std::uint8_t* bits_out, std::int64_t* stats) {
  return guarded([&] {
    const vitdec::Trellis t = vitdec::build_trellis(make_spec(k, b, polys));
    const vitdec::LlrBlock block = Eigen::Map<const vitdec::LlrBlock>(llr, b, n);
    put_out(vitdec::framed_decode(block, t, make_cfg(f, v1, v2, f0, start, seed), workers), bits_out, stats);
  });
}

/// Same, int8 input fed to the reference as double(q) (SURVEY §8(c) protocol).
int vdref_framed_decode_i8(int k, int b, const std::uint32_t* polys, const std::int8_t* llr, std::int64_t n,
                           int f, int v1, int v2, int f0, int start, std::uint64_t seed, int workers,
                           std::uint8_t* bits_out, std::int64_t* stats) {
  return guarded([&] {
    const vitdec::Trellis t = vitdec::build_trellis(make_spec(k, b, polys));
    vitdec::LlrBlock block(b, n);
    for (std::int64_t i = 0; i < n * b; ++i) block.data()[i] = static_cast<double>(llr[i]);
    put_out(vitdec::framed_decode(block, t, make_cfg(f, v1, v2, f0, start, seed), workers), bits_out, stats);
  });
}

int vdref_serial_decode_f64(int k, int b, const std::uint32_t* polys, const double* llr, std::int64_t n,
                            std::uint8_t* bits_out, std::int64_t* stats) {
  return guarded([&] {
    const vitdec::Trellis t = vitdec::build_trellis(make_spec(k, b, polys));
    const vitdec::LlrBlock block = Eigen::Map<const vitdec::LlrBlock>(llr, b, n);
    put_out(vitdec::serial_decode(block, t), bits_out, stats);
  });
}

/// The throughput-bench data recipe (reference berlab.cpp:138-142): n info
/// bits from random_bits(n, mix_seed(seed,1)), encoded, BPSK, AWGN at the
/// base-rate sigma for ebn0_db with seed mix_seed(seed,2). Writes the n*B
/// received stream and the n sent bits.
int vdref_gen_bench_block(int k, int b, const std::uint32_t* polys, std::int64_t n, double ebn0_db,
                          std::uint64_t seed, double* rx_out, std::uint8_t* sent_out) {
  return guarded([&] {
    const vitdec::CodeSpec spec = make_spec(k, b, polys);
    const vitdec::Trellis t = vitdec::build_trellis(spec);
    const vitdec::BitVec sent = vitdec::random_bits(static_cast<std::size_t>(n), vitdec::mix_seed(seed, 1));
    const double sigma = vitdec::sigma_from_ebn0(ebn0_db, spec.base_rate());
    const Eigen::ArrayXd rx = vitdec::awgn(vitdec::modulate_bpsk(vitdec::encode(sent, t)), sigma,
                                           vitdec::mix_seed(seed, 2));
    std::memcpy(rx_out, rx.data(), sizeof(double) * rx.size());
    std::memcpy(sent_out, sent.data(), sent.size());
  });
}

/// One block of the BER-sweep recipe (reference berlab.cpp:66-80),
/// unpunctured: block_seed as computed by run_ber_sweep.
int vdref_gen_sweep_block(int k, int b, const std::uint32_t* polys, std::int64_t n, double sigma,
                          std::uint64_t block_seed, double* rx_out, std::uint8_t* sent_out) {
  return guarded([&] {
    const vitdec::CodeSpec spec = make_spec(k, b, polys);
    const vitdec::Trellis t = vitdec::build_trellis(spec);
    const vitdec::BitVec sent = vitdec::random_bits(static_cast<std::size_t>(n), vitdec::mix_seed(block_seed, 1));
    const Eigen::ArrayXd rx = vitdec::awgn(vitdec::modulate_bpsk(vitdec::encode(sent, t)), sigma,
                                           vitdec::mix_seed(block_seed, 2));
    std::memcpy(rx_out, rx.data(), sizeof(double) * rx.size());
    std::memcpy(sent_out, sent.data(), sent.size());
  });
}

/// Reference run_ber_sweep (serial decoder when f == 0). errors_out/bits_out
/// receive one entry per Eb/N0 point.
int vdref_ber_sweep(int k, int b, const std::uint32_t* polys, const char* pattern, int f, int v1, int v2, int f0,
                    int start, std::uint64_t frame_seed, int hard, const double* ebn0, int npoints,
                    std::int64_t bits_per_point, std::int64_t block_bits, std::uint64_t seed, int workers,
                    std::int64_t* errors_out, std::int64_t* bits_out) {
  return guarded([&] {
    vitdec::SweepSetup s;
    s.spec = make_spec(k, b, polys);
    s.pattern = vitdec::PuncturePattern::named(pattern);
    if (f > 0) s.frame = make_cfg(f, v1, v2, f0, start, frame_seed);
    s.hard = hard != 0;
    s.ebn0_db.assign(ebn0, ebn0 + npoints);
    s.bits_per_point = bits_per_point;
    s.block_bits = block_bits;
    s.seed = seed;
    s.workers = workers;
    const auto pts = vitdec::run_ber_sweep(s);
    for (std::size_t i = 0; i < pts.size(); ++i) {
      errors_out[i] = pts[i].errors;
      bits_out[i] = pts[i].bits;
    }
  });
}

/// Reference depuncture of a punctured double stream; writes B x stages.
int vdref_depuncture(const char* pattern, const double* punctured, std::int64_t len, double* out,
                     std::int64_t out_cap, std::int64_t* stages_out) {
  return guarded([&] {
    const vitdec::PuncturePattern p = vitdec::PuncturePattern::named(pattern);
    Eigen::ArrayXd stream(len);
    for (std::int64_t i = 0; i < len; ++i) stream[i] = punctured[i];
    const vitdec::LlrBlock block = vitdec::depuncture(stream, p);
    *stages_out = block.cols();
    if (block.size() > out_cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, block.data(), sizeof(double) * block.size());
  });
}

}  // extern "C"
