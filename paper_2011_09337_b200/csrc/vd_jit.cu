// Run-time instantiation of the fast kernel for codes outside the
// precompiled list (vd_fast_k*.cu): any rate-1/2, 1/3 or 1/4 code with
// 5 <= K <= 10 (complement-paired, reference Trellis::complement_paired,
// trellis.cpp:93-100, or not). The kernel bakes the polynomials into compile-time
// table selections (vd_fast_dev.cuh, Geo::xreg / xlane), so a new code needs
// a new instantiation: NVRTC compiles vd_fast_dev.cuh (embedded in this
// library at build time) for sm_100a, the cubin is loaded with the runtime's
// library API and cached per process and on disk.
//
//   VITDEC_JIT=0          disable (such codes then use the generic kernel)
//   VITDEC_JIT_CACHE=DIR  cubin cache directory (default ~/.cache/vitdec_b200/jit;
//                         "" or "0": no disk cache)
//
// NVRTC is opened with dlopen on first use, so the library loads (and the
// precompiled codes run) without it; codes that would need it then use the
// generic kernel.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "vd_internal.h"

namespace vd {
namespace jit {
namespace {

// Sources the kernel needs, embedded by the Makefile (build/vd_jit_sources.inc
// defines kJitHeaders[] = {{"name", "text"}, ...}).
struct Src {
  const char* name;
  const char* text;
};
#include "vd_jit_sources.inc"

// NVRTC entry points (dlopen'ed).
typedef int (*CreateFn)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*DestroyFn)(void**);
typedef int (*CompileFn)(void*, int, const char* const*);
typedef int (*SizeFn)(void*, std::size_t*);
typedef int (*GetFn)(void*, char*);
typedef int (*AddNameFn)(void*, const char*);
typedef int (*LoweredFn)(void*, const char*, const char**);
struct Nvrtc {
  bool ok = false;
  CreateFn create;
  DestroyFn destroy;
  CompileFn compile;
  SizeFn log_size, cubin_size;
  GetFn log, cubin;
  AddNameFn add_name;
  LoweredFn lowered;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* lib : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      if ((h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    }
    if (!h) return r;
    r.create = reinterpret_cast<CreateFn>(dlsym(h, "nvrtcCreateProgram"));
    r.destroy = reinterpret_cast<DestroyFn>(dlsym(h, "nvrtcDestroyProgram"));
    r.compile = reinterpret_cast<CompileFn>(dlsym(h, "nvrtcCompileProgram"));
    r.log_size = reinterpret_cast<SizeFn>(dlsym(h, "nvrtcGetProgramLogSize"));
    r.log = reinterpret_cast<GetFn>(dlsym(h, "nvrtcGetProgramLog"));
    r.cubin_size = reinterpret_cast<SizeFn>(dlsym(h, "nvrtcGetCUBINSize"));
    r.cubin = reinterpret_cast<GetFn>(dlsym(h, "nvrtcGetCUBIN"));
    r.add_name = reinterpret_cast<AddNameFn>(dlsym(h, "nvrtcAddNameExpression"));
    r.lowered = reinterpret_cast<LoweredFn>(dlsym(h, "nvrtcGetLoweredName"));
    r.ok = r.create && r.destroy && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.add_name &&
           r.lowered;
    return r;
  }();
  return n;
}

thread_local std::string t_log;

std::uint64_t fnv1a(const std::string& s, std::uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  const char* env = std::getenv("VITDEC_JIT_CACHE");
  if (env) return (env[0] == '\0' || std::strcmp(env, "0") == 0) ? std::string() : std::string(env);
  const char* home = std::getenv("HOME");
  if (!home || !home[0]) return std::string();
  return std::string(home) + "/.cache/vitdec_b200/jit";
}

void mkdirs(const std::string& dir) {
  for (std::size_t i = 1; i <= dir.size(); ++i) {
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  }
}

bool read_file(const std::string& path, std::string* out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  *out = ss.str();
  return !out->empty();
}

// Compiles `expr` (an address-of expression naming the kernel instantiation);
// returns the cubin and the lowered (mangled) kernel name.
bool compile(const std::string& expr, std::string* cubin, std::string* name) {
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    t_log = "NVRTC (libnvrtc.so.12) not found";
    return false;
  }
  std::vector<const char*> hdr_text, hdr_name;
  for (const Src& s : kJitHeaders) {
    hdr_text.push_back(s.text);
    hdr_name.push_back(s.name);
  }
  const std::string src = "#include \"vd_fast_dev.cuh\"\n#include \"vd_small_dev.cuh\"\n";
  void* prog = nullptr;
  if (nv.create(&prog, src.c_str(), "vd_jit_fast.cu", static_cast<int>(hdr_text.size()), hdr_text.data(),
                hdr_name.data()) != 0) {
    t_log = "nvrtcCreateProgram failed";
    return false;
  }
  nv.add_name(prog, expr.c_str());
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "-DVD_JIT=1"};
  const int rc = nv.compile(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  std::size_t ls = 0;
  nv.log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls) nv.log(prog, &log[0]);
  bool ok = rc == 0;
  if (ok) {
    const char* lowered = nullptr;
    std::size_t cs = 0;
    ok = nv.lowered(prog, expr.c_str(), &lowered) == 0 && lowered && nv.cubin_size(prog, &cs) == 0 && cs > 0;
    if (ok) {
      *name = lowered;
      cubin->assign(cs, '\0');
      ok = nv.cubin(prog, &(*cubin)[0]) == 0;
    }
  }
  if (!ok) t_log = "NVRTC compile of " + expr + " failed: " + log.substr(0, 4000);
  nv.destroy(&prog);
  return ok;
}

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};

}  // namespace

bool enabled() {
  const char* e = std::getenv("VITDEC_JIT");
  if (e && std::strcmp(e, "0") == 0) return false;
  // without NVRTC on this machine the codes keep the generic kernel
  return nvrtc().ok;
}

const std::string& last_log() { return t_log; }

const void* kernel(const std::string& expr, cudaError_t* err);

std::string code_type(int k, int b, const std::uint32_t* polys) {
  char buf[160];
  std::snprintf(buf, sizeof(buf), "vd::fast::CodeB<%d, %d, %uu, %uu, %uu, %uu>", k, b, polys[0], polys[1],
                b > 2 ? polys[2] : 0u, b > 3 ? polys[3] : 0u);
  return buf;
}

std::string expression(int k, int b, const std::uint32_t* polys, bool tm, bool gl) {
  return "&vd::fast::fast_kernel<" + code_type(k, b, polys) + ", 16, " + (tm ? "true" : "false") + ", " +
         (gl ? "true" : "false") + ">";
}

bool compile_check(int k, int b, const std::uint32_t* polys) {
  std::string cubin, name;
  return compile(expression(k, b, polys, true, false), &cubin, &name);
}

const void* fast_kernel(int k, int b, const std::uint32_t* polys, bool tm, bool gl, cudaError_t* err) {
  return kernel(expression(k, b, polys, tm, gl), err);
}

const void* punct_kernel(int k, const std::uint32_t* polys, int pattern, cudaError_t* err) {
  if (pattern != 23 && pattern != 34) return nullptr;
  return kernel("&vd::fast::fast_kernel<" + code_type(k, 2, polys) + ", 16, true, false, vd::fast::PunctR" +
                    std::to_string(pattern) + ">",
                err);
}

const void* small_kernel(int k, const std::uint32_t* polys, cudaError_t* err) {
  return kernel("&vd::fast::small_kernel<" + code_type(k, 2, polys) + ", 8>", err);
}

const void* kernel(const std::string& expr, cudaError_t* err) {
  static std::mutex mu;
  static std::map<std::string, Entry> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(expr);
  if (it != cache.end()) return reinterpret_cast<const void*>(it->second.kern);
  // disk cache: keyed by the embedded sources + options + instantiation
  std::string key = expr;
  for (const Src& s : kJitHeaders) key += s.text;
  char hex[32];
  std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(fnv1a(key)));
  const std::string dir = cache_dir();
  const std::string path = dir.empty() ? std::string() : dir + "/" + hex + ".cubin";
  const std::string name_path = dir.empty() ? std::string() : dir + "/" + hex + ".name";
  std::string cubin, name;
  if (path.empty() || !read_file(path, &cubin) || !read_file(name_path, &name)) {
    if (!compile(expr, &cubin, &name)) {
      *err = cudaErrorInvalidSource;
      return nullptr;
    }
    if (!path.empty()) {
      mkdirs(dir);
      const std::string tmp = path + "." + std::to_string(getpid());
      std::ofstream(tmp, std::ios::binary).write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
      std::ofstream(name_path + "." + std::to_string(getpid()), std::ios::binary) << name;
      std::rename((name_path + "." + std::to_string(getpid())).c_str(), name_path.c_str());
      std::rename(tmp.c_str(), path.c_str());
    }
  }
  Entry e;
  cudaError_t ce = cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (ce == cudaSuccess) ce = cudaLibraryGetKernel(&e.kern, e.lib, name.c_str());
  if (ce != cudaSuccess) {
    t_log = "loading the JIT cubin of " + expr + ": " + cudaGetErrorString(ce);
    *err = ce;
    return nullptr;
  }
  cache[expr] = e;
  return reinterpret_cast<const void*>(e.kern);
}

}  // namespace jit
}  // namespace vd
