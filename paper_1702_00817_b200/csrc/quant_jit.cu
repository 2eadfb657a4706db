// quant_jit.cu — run-time specialisation of the quantised kernels for one
// quantiser table.
//
// The generic kernels read the 64 per-position constants from the kernel
// parameters (2 LDC.64 + 1 LDCU per position per unit: ~7.5 % of the quant
// kernel's instructions).  A kernel compiled with the table as compile-time
// constants turns them into instruction immediates (+5.5 % on config 4,
// DESIGN.md §4).  Tables are runtime data, so the specialised kernel is built
// here with NVRTC from the same headers (embedded at build time), once a table
// has been used ADCT_QUANT_JIT_AFTER times (default 3; 0 disables), and cached
// for the life of the process.  NVRTC is dlopen'ed and the driver API is
// reached through cudaGetDriverEntryPoint, so the library links nothing new;
// when either is missing, or a compile fails, the generic kernel keeps
// running (it is the same GPU computation, bit for bit).
#include "adct_jit.h"

#include <cuda.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "adct_jit_src.inc"  // kJitDeviceH, kJitKernelsH (generated from the headers by the Makefile)

namespace adct {
namespace jit {
namespace {

typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;

struct Nvrtc {
  bool ok = false;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*add_name)(nvrtcProgram, const char*);
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*lowered)(nvrtcProgram, const char*, const char**);
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*);
  nvrtcResult (*cubin)(nvrtcProgram, char*);
  nvrtcResult (*log_size)(nvrtcProgram, size_t*);
  nvrtcResult (*log)(nvrtcProgram, char*);
  nvrtcResult (*destroy)(nvrtcProgram*);
};

struct Driver {
  bool ok = false;
  CUresult (*load)(CUmodule*, const void*);
  CUresult (*get_function)(CUfunction*, CUmodule, const char*);
  CUresult (*set_attribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**);
};

struct Entry {
  int uses = 0;
  int state = 0;  // 0 generic, 1 specialised, 2 being built (by another thread), -1 specialisation failed
  CUfunction fn = nullptr;
};

// Tables that are used fewer than the threshold times keep an entry (a use
// count); past this many entries the never-specialised ones are dropped.
constexpr size_t kMaxEntries = 256;

std::mutex g_mu;
std::map<std::string, Entry> g_cache;
std::atomic<long long> g_compiled{0}, g_launches{0}, g_failures{0};

int threshold() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_QUANT_JIT_AFTER");
    return e ? std::atoi(e) : 3;
  }();
  return v;
}

Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (h == nullptr) return r;
#define ADCT_SYM(field, name)                                           \
  r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, name));        \
  if (r.field == nullptr) return r;
    ADCT_SYM(create, "nvrtcCreateProgram")
    ADCT_SYM(add_name, "nvrtcAddNameExpression")
    ADCT_SYM(compile, "nvrtcCompileProgram")
    ADCT_SYM(lowered, "nvrtcGetLoweredName")
    ADCT_SYM(cubin_size, "nvrtcGetCUBINSize")
    ADCT_SYM(cubin, "nvrtcGetCUBIN")
    ADCT_SYM(log_size, "nvrtcGetProgramLogSize")
    ADCT_SYM(log, "nvrtcGetProgramLog")
    ADCT_SYM(destroy, "nvrtcDestroyProgram")
#undef ADCT_SYM
    r.ok = true;
    return r;
  }();
  return n;
}

Driver& driver() {
  static Driver d = [] {
    Driver r;
#define ADCT_DRV(field, name)                                                                 \
  {                                                                                           \
    void* fp = nullptr;                                                                       \
    cudaDriverEntryPointQueryResult st;                                                       \
    if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &st) != cudaSuccess ||          \
        st != cudaDriverEntryPointSuccess || fp == nullptr)                                   \
      return r;                                                                               \
    r.field = reinterpret_cast<decltype(r.field)>(fp);                                        \
  }
    ADCT_DRV(load, "cuModuleLoadData")
    ADCT_DRV(get_function, "cuModuleGetFunction")
    ADCT_DRV(set_attribute, "cuFuncSetAttribute")
    ADCT_DRV(launch, "cuLaunchKernel")
#undef ADCT_DRV
    r.ok = true;
    return r;
  }();
  return d;
}

const char* kernel_expression(int kind) {
  switch (kind) {
    case kQuantPairAligned: return "adct::k_quant_p<true, false, BakedTab>";
    case kQuantPairFlip: return "adct::k_quant_p<true, true, BakedTab>";
    case kQuantSingleAligned: return "adct::k_quant_p<false, false, BakedTab>";
    case kQuantSingleFlip: return "adct::k_quant_p<false, true, BakedTab>";
    case kHybrid: return "adct::k_quant_hybrid<BakedTab>";
    case kQuantPairAligned + kFloatOffset: return "adct::k_quant_p<true, false, BakedTab, true>";
    case kQuantPairFlip + kFloatOffset: return "adct::k_quant_p<true, true, BakedTab, true>";
    case kQuantSingleAligned + kFloatOffset: return "adct::k_quant_p<false, false, BakedTab, true>";
    case kQuantSingleFlip + kFloatOffset: return "adct::k_quant_p<false, true, BakedTab, true>";
    case kHybridF: return "adct::k_quant_hybrid<BakedTab, true>";
    default: return nullptr;
  }
}

std::string baked_source(const QParamsDev& q) {
  std::string s = "#include \"adct_kernels.cuh\"\nstruct BakedTab {\n  static constexpr bool kBaked = true;\n";
  s += "  static __device__ __forceinline__ uint4 pos(const adct::QParamsDev&, int p) {\n";
  s += "    constexpr unsigned t[64][4] = {";
  char buf[96];
  for (int p = 0; p < 64; ++p) {
    std::snprintf(buf, sizeof buf, "%s{%uu,%uu,%uu,%uu}", p ? "," : "", q.pos[p].x, q.pos[p].y, q.pos[p].z,
                  q.pos[p].w);
    s += buf;
  }
  s += "};\n    return make_uint4(t[p][0], t[p][1], t[p][2], t[p][3]);\n  }\n";
  s += "  static __device__ __forceinline__ unsigned wadd(const adct::QParamsDev&, int p) {\n";
  s += "    constexpr unsigned t[64] = {";
  for (int p = 0; p < 64; ++p) {
    std::snprintf(buf, sizeof buf, "%s%uu", p ? "," : "", q.wadd[p]);
    s += buf;
  }
  s += "};\n    return t[p];\n  }\n};\n";
  return s;
}

CUfunction build(int kind, const QParamsDev& q) {
  Nvrtc& nv = nvrtc();
  Driver& dr = driver();
  if (!nv.ok || !dr.ok) return nullptr;
  const std::string src = baked_source(q);
  const char* headers[] = {kJitDeviceH, kJitKernelsH};
  const char* names[] = {"adct_device.cuh", "adct_kernels.cuh"};
  nvrtcProgram prog = nullptr;
  if (nv.create(&prog, src.c_str(), "adct_quant_jit.cu", 2, headers, names) != 0) return nullptr;
  const char* expr = kernel_expression(kind);
  CUfunction fn = nullptr;
  bool good = expr != nullptr && nv.add_name(prog, expr) == 0;
  // ADCT_JIT_OPTS: one extra NVRTC option (e.g. --maxrregcount=120) for A/B runs
  const char* extra = std::getenv("ADCT_JIT_OPTS");
  if (extra != nullptr && *extra == '\0') extra = nullptr;  // set but empty: no extra option
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", extra ? extra : ""};
  if (good && nv.compile(prog, extra ? 4 : 3, opts) != 0) {
    good = false;
    if (std::getenv("ADCT_QUANT_JIT_LOG")) {
      size_t n = 0;
      nv.log_size(prog, &n);
      std::vector<char> log(n + 1, 0);
      nv.log(prog, log.data());
      std::fprintf(stderr, "adct quant JIT compile failed:\n%s\n", log.data());
    }
  }
  const char* lowered = nullptr;
  size_t n = 0;
  if (good) good = nv.lowered(prog, expr, &lowered) == 0 && nv.cubin_size(prog, &n) == 0 && n > 0;
  std::vector<char> cubin(n);
  if (good) good = nv.cubin(prog, cubin.data()) == 0;
  CUmodule mod = nullptr;
  if (good) good = dr.load(&mod, cubin.data()) == CUDA_SUCCESS;  // module lives for the process
  if (good) good = dr.get_function(&fn, mod, lowered) == CUDA_SUCCESS;
  const int smem = (kind == kHybrid || kind == kHybridF) ? (int)kHybridSmem : (int)(2 * 8 * kThreads * sizeof(uint4));
  if (good)
    good = dr.set_attribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem) == CUDA_SUCCESS;
  nv.destroy(&prog);
  return good ? fn : nullptr;
}

}  // namespace

void* quant_function(int kind, const QParamsDev& q, cudaStream_t stream) {
  const int after = threshold();
  if (after <= 0) return nullptr;
  // never build while `stream` is being captured into a CUDA graph (module
  // loading is not a capturable operation); a kernel built earlier is fine
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
  int dev = 0;  // a loaded module belongs to one device's context: key by device too
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::string key(reinterpret_cast<const char*>(&q), sizeof(QParamsDev));
  key.push_back((char)kind);
  key.append(reinterpret_cast<const char*>(&dev), sizeof dev);
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
      if (g_cache.size() >= kMaxEntries)
        for (auto jt = g_cache.begin(); jt != g_cache.end();)
          jt = jt->second.state == 0 ? g_cache.erase(jt) : std::next(jt);
      it = g_cache.emplace(key, Entry{}).first;
    }
    Entry& e = it->second;
    if (e.state == 1) return e.fn;
    if (e.state != 0 || capturing) return nullptr;  // failed, or another thread is compiling it
    if (++e.uses < after) return nullptr;
    e.state = 2;  // this thread compiles; others keep launching the generic kernel meanwhile
  }
  // NVRTC + module load outside the lock: other tables and devices are not
  // held up for the seconds a compile takes
  CUfunction fn = build(kind, q);
  std::lock_guard<std::mutex> lock(g_mu);
  Entry& e = g_cache[key];
  e.fn = fn;
  e.state = fn ? 1 : -1;
  (fn ? g_compiled : g_failures)++;
  return fn;
}

int launch(void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, void** args) {
  Driver& dr = driver();
  if (!dr.ok) return (int)CUDA_ERROR_NOT_INITIALIZED;
  g_launches++;
  return (int)dr.launch(reinterpret_cast<CUfunction>(fn), grid.x, grid.y, grid.z, block.x, block.y, block.z,
                        (unsigned)smem, reinterpret_cast<CUstream>(stream), args, nullptr);
}

void stats(long long* compiled, long long* launches, long long* failures) {
  if (compiled) *compiled = g_compiled.load();
  if (launches) *launches = g_launches.load();
  if (failures) *failures = g_failures.load();
}

}  // namespace jit
}  // namespace adct
