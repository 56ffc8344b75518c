// mgp_abi.cu -- extern "C" entry points of libmgp.so (see include/megopolis_b200.h).
//
// Host-side responsibilities: argument validation with the reference's error texts
// (pkg/src/megores/resample.py:84-108, weights.py:114-131), kernel selection, the
// Megopolis offsets (computed on the host like M/resample.py:263-265 and carried to
// the device in the kernel parameter space), stream-ordered scratch, and the
// host-buffer path that overlaps ancestor download with compute.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#ifndef MGP_COPY_NT
#define MGP_COPY_NT 1
#endif

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <curand_philox4x32_x.h>

#include "megopolis_b200.h"
#include "mgp_kernels.cuh"
#include "mgp_prefix.cuh"

using namespace mgp;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_err(cudaError_t e, const char* what) {
  return set_err((int)e, "CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
}

#define CUDA_TRY(x)                                   \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) return cuda_err(e_, #x);   \
  } while (0)

#define LAUNCH_CHECK(what)                                  \
  do {                                                      \
    cudaError_t e_ = cudaGetLastError();                    \
    if (e_ != cudaSuccess) return cuda_err(e_, what);       \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline uint32_t ilog2(uint64_t v) { uint32_t r = 0; while ((1ull << r) < v) ++r; return r; }

constexpr int64_t MAX_N = (1ll << 31) - 1;

int check_common(int dtype, int64_t n, int32_t b, int rng) {
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64, got %d", dtype);
  if (rng != MGP_RNG_MEGORES && rng != MGP_RNG_PHILOX) return set_err(MGP_EINVAL, "unknown rng stream %d", rng);
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N=%lld exceeds this build's limit of 2^31-1 particles", (long long)n);
  if (b < 1) return set_err(MGP_EINVAL, "B must be >= 1, got %d", b);
  return 0;
}

int check_warp(int64_t n, int32_t warp, int strict, const char* name) {  // M/resample.py:59-75, 103-108
  if (warp < 1) return set_err(MGP_EINVAL, "warp_size must be positive, got %d", warp);
  if (strict && n % warp)
    return set_err(MGP_EINVAL, "%s requires N (%lld) to be a multiple of the warp size (%d) in strict mode", name,
                   (long long)n, warp);
  return 0;
}

int check_partition(int64_t n, int32_t part_bytes, int64_t* n_w, int64_t* n_part) {  // M/resample.py:84-93
  if (part_bytes < 1 || part_bytes % 4) return set_err(MGP_EINVAL, "partition_bytes must be a positive multiple of word_bytes");
  *n_w = part_bytes / 4;
  if (n % *n_w) return set_err(MGP_EINVAL, "N=%lld is not divisible by the partition width %lld", (long long)n, (long long)*n_w);
  *n_part = n / *n_w;
  return 0;
}

// ---------------------------------------------------------------------------
// Stream-ordered scratch from a private per-device memory pool.  The pool keeps freed
// blocks (release threshold UINT64_MAX), so the per-call allocation of reduction heaps,
// offsets and the host-path buffers is a pool hit instead of a remap after every
// synchronisation.  It is the library's own pool: the device's default pool (and with it
// the host application's cudaMallocAsync behaviour) is never modified.
// mgp_release_cached_memory() trims it.

std::mutex g_pool_mu;
std::vector<std::pair<int, cudaMemPool_t>> g_pools;

cudaError_t lib_pool(cudaMemPool_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto& dp : g_pools)
    if (dp.first == dev) { *out = dp.second; return cudaSuccess; }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
  uint64_t thr = UINT64_MAX;
  if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess) return e;
  g_pools.emplace_back(dev, pool);
  *out = pool;
  return cudaSuccess;
}

// cudaMallocAsync from the library's pool on the current device
template <typename T>
cudaError_t pool_malloc(T** out, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool;
  cudaError_t e = lib_pool(&pool);
  if (e != cudaSuccess) return e;
  void* q = nullptr;
  e = cudaMallocFromPoolAsync(&q, bytes ? bytes : 1, pool, st);
  *out = static_cast<T*>(q);
  return e;
}

// Stream-ordered scratch owned by one call: every block allocated through it is released
// (cudaFreeAsync, ordered after the work queued so far) when it goes out of scope, so the
// early returns of CUDA_TRY / LAUNCH_CHECK do not leak.
class Scratch {
 public:
  explicit Scratch(cudaStream_t st) : st_(st) {}
  ~Scratch() {
    for (auto it = p_.rbegin(); it != p_.rend(); ++it) cudaFreeAsync(*it, st_);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <typename T>
  cudaError_t alloc(T** out, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = pool_malloc(&q, bytes, st_);
    if (e == cudaSuccess) p_.push_back(q);
    *out = static_cast<T*>(q);
    return e;
  }

 private:
  cudaStream_t st_;
  std::vector<void*> p_;
};

// ---------------------------------------------------------------------------
// pairwise reduction plumbing

int pw_depth(int64_t n) {
  std::vector<int64_t> sizes{n}, next;
  int d = 0;
  for (;;) {
    int64_t mx = 0;
    for (int64_t s : sizes) mx = s > mx ? s : mx;
    if (mx <= PW_CHUNK) return d;
    next.clear();
    for (int64_t s : sizes) {
      int64_t n2 = s / 2;
      n2 -= n2 % 8;
      next.push_back(n2);
      next.push_back(s - n2);
    }
    std::sort(next.begin(), next.end());
    next.erase(std::unique(next.begin(), next.end()), next.end());
    sizes.swap(next);
    ++d;
  }
}

template <class Elem, typename WT, bool STATS>
int pw_reduce(const Elem& e, const WT* wraw, int64_t n, PwOut out, cudaStream_t st) {
  Scratch sc(st);
  const int depth = pw_depth(n);
  const int64_t nch = 1ll << depth;
  double* heap = nullptr;
  WStats* cst = nullptr;
  CUDA_TRY(sc.alloc(&heap, sizeof(double) * 2 * nch));
  if (STATS) CUDA_TRY(sc.alloc(&cst, sizeof(WStats) * nch));
  if (n == (int64_t)PW_CHUNK << depth)  // power-of-two N >= 4096: perfect 32-leaf chunk subtrees
    k_pw_chunks4096<Elem, WT, STATS><<<(unsigned)nch, PW_THREADS, 0, st>>>(e, wraw, depth, heap, cst);
  else
    k_pw_chunks<Elem, WT, STATS><<<(unsigned)nch, PW_THREADS, 0, st>>>(e, wraw, n, depth, heap, cst);
  LAUNCH_CHECK("k_pw_chunks");
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = MGP_PW_PDL;
  cudaLaunchConfig_t la{};
  la.gridDim = dim3(1);
  la.blockDim = dim3(1024);
  la.stream = st;
  la.attrs = at;
  la.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&la, k_pw_final, heap, depth, n, (const WStats*)cst, out));
  return 0;
}

// ---------------------------------------------------------------------------
// host offsets

void offsets_host(uint64_t seed, int64_t n, int32_t b, int rng, int64_t* out) {
  const uint64_t base = megores_base(seed);
  for (int32_t t = 0; t < b; ++t) {
    if (rng == MGP_RNG_MEGORES) out[t] = below_from_hash(mix64(megores_key(base, GLOBAL_OFFSET_LANE, (uint64_t)t)), n);
    else out[t] = below_from_word(p4_word(philox_block(seed, GLOBAL_OFFSET_LANE, (uint64_t)t >> 2), t & 3), n);
  }
}

// ---------------------------------------------------------------------------
// kernel dispatch helpers

// Particles per thread: 4 for the Philox stream (interleaved Philox chains; measured 5.97 -> 5.54 ms
// at 2^24, PPT 1 -> 4; scripts/mb/ppt_sweep.sh),
// 1 for megores (its issue-bound splitmix chain gains nothing from more ILP: 2 or 4 particles
// per thread, with or without the half split, measured 0.6-0.8% slower; scripts/mb/ppt_megores.sh).
#ifndef MGP_PPT_PHILOX
#define MGP_PPT_PHILOX 4
#endif
#ifndef MGP_PPT_MEGORES
#define MGP_PPT_MEGORES 1
#endif

template <int RNG>
constexpr int mego_ppt() { return RNG == RNG_PHILOX ? MGP_PPT_PHILOX : MGP_PPT_MEGORES; }

template <int RNG, typename WT, bool POW2, bool NZ, bool TEX>
int launch_mego_w32(const ResampleArgs& a, const OffChunk& oc, cudaStream_t st) {
  const unsigned grid = (unsigned)((a.p_end - a.p0 + RS_THREADS - 1) / RS_THREADS);
  constexpr int PPT = mego_ppt<RNG>();
  if constexpr (POW2 && PPT == 4) {
    // N = 2^k >= 256, full range or an explicit lower-half range (a.half): the half-split
    // variant (j(i + N/2) = j(i) ^ N/2); particles i and i + N/2 for i in [p0, p_end)
    if (a.half || (a.p0 == 0 && a.p_end == a.n && a.n >= 256)) {
      ResampleArgs h = a;
      if (!a.half) { h.p0 = 0; h.p_end = a.n / 2; }
      const unsigned hgrid = (unsigned)((h.p_end - h.p0) / 128);
      if (hgrid == 0) return 0;
      if (a.rows_out) {
        k_megopolis_w32<RNG, WT, POW2, NZ, TEX, PPT, true, true><<<hgrid, RS_THREADS / PPT, 0, st>>>(h, oc);
      } else if constexpr (RNG == RNG_PHILOX && sizeof(WT) == 4 && NZ && TEX) {
        k_megopolis_philox_half<<<hgrid, 64, 0, st>>>(h, oc);  // the headline configuration
      } else {
        k_megopolis_w32<RNG, WT, POW2, NZ, TEX, PPT, true><<<hgrid, RS_THREADS / PPT, 0, st>>>(h, oc);
      }
      LAUNCH_CHECK("k_megopolis_w32");
      return 0;
    }
  }
  if constexpr (RNG == RNG_MEGORES && sizeof(WT) == 4 && NZ && TEX) {
    // the reference's stream on float32 weights: float32 bracket + exact fallback
    if (a.rows_out) k_megopolis_megores_f32<POW2, true><<<grid, RS_THREADS, 0, st>>>(a, oc);
    else k_megopolis_megores_f32<POW2><<<grid, RS_THREADS, 0, st>>>(a, oc);
    LAUNCH_CHECK("k_megopolis_megores_f32");
    return 0;
  }
  if (a.rows_out) k_megopolis_w32<RNG, WT, POW2, NZ, TEX, PPT, false, true><<<grid, RS_THREADS / PPT, 0, st>>>(a, oc);
  else k_megopolis_w32<RNG, WT, POW2, NZ, TEX, PPT><<<grid, RS_THREADS / PPT, 0, st>>>(a, oc);
  LAUNCH_CHECK("k_megopolis_w32");
  return 0;
}

template <int RNG, typename WT>
int dispatch_mego_w32(const ResampleArgs& a, const OffChunk& oc, bool pow2, bool nz, cudaStream_t st) {
#define MEGO_CASE(P, Z, T)                                                    \
  if (pow2 == P && nz == Z && (a.tex != 0) == T) {                            \
    if constexpr (!T || sizeof(WT) == 4) return launch_mego_w32<RNG, WT, P, Z, T>(a, oc, st); \
  }
  MEGO_CASE(true, true, true)
  MEGO_CASE(true, false, true)
  MEGO_CASE(false, true, true)
  MEGO_CASE(false, false, true)
  MEGO_CASE(true, true, false)
  MEGO_CASE(true, false, false)
  MEGO_CASE(false, true, false)
  MEGO_CASE(false, false, false)
#undef MEGO_CASE
  return set_err(MGP_EINVAL, "internal: no megopolis variant");
}

template <int RNG, typename WT, bool POW2, bool NZ>
int launch_metro(const ResampleArgs& a, cudaStream_t st) {
  const unsigned grid = (unsigned)((a.p_end - a.p0 + RS_THREADS - 1) / RS_THREADS);
  k_metropolis<RNG, WT, POW2, NZ><<<grid, RS_THREADS, 0, st>>>(a);
  LAUNCH_CHECK("k_metropolis");
  return 0;
}

template <int RNG, typename WT>
int dispatch_metro(const ResampleArgs& a, bool pow2, bool nz, cudaStream_t st) {
  if (nz) return pow2 ? launch_metro<RNG, WT, true, true>(a, st) : launch_metro<RNG, WT, false, true>(a, st);
  return pow2 ? launch_metro<RNG, WT, true, false>(a, st) : launch_metro<RNG, WT, false, false>(a, st);
}

constexpr int C1_SMEM_MAX = 96 * 1024;

template <int RNG, typename WT, bool POW2, bool NZ, bool C2, bool STAGE>
int launch_c12(const ResampleArgs& a, cudaStream_t st) {
  const unsigned grid = (unsigned)((a.p_end - a.p0 + RS_THREADS - 1) / RS_THREADS);
  size_t smem = STAGE ? (size_t)(RS_THREADS / 32) * a.n_w * sizeof(WT) : 0;
  auto kern = k_c12_w32<RNG, WT, POW2, NZ, C2, STAGE>;
  if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, RS_THREADS, smem, st>>>(a);
  LAUNCH_CHECK("k_c12_w32");
  return 0;
}

template <int RNG, typename WT, bool C2>
int dispatch_c12(const ResampleArgs& a, bool pow2, bool nz, bool no_stage, cudaStream_t st) {
  const bool stage = !C2 && !no_stage && (size_t)(RS_THREADS / 32) * a.n_w * sizeof(WT) <= (size_t)C1_SMEM_MAX;
#define C12_CASE(P, Z)                                                        \
  if (pow2 == P && nz == Z) {                                                 \
    if (stage) return launch_c12<RNG, WT, P, Z, C2, !C2>(a, st);              \
    return launch_c12<RNG, WT, P, Z, C2, false>(a, st);                       \
  }
  C12_CASE(true, true)
  C12_CASE(false, true)
  C12_CASE(true, false)
  C12_CASE(false, false)
#undef C12_CASE
  return set_err(MGP_EINVAL, "internal: no c1/c2 variant");
}

// ---------------------------------------------------------------------------
// float32 weights as a 1-D linear texture: the texture unit does the partner-address
// arithmetic.  Objects are cached per (device, pointer, length) in a bounded LRU.  A
// lookup pins its entry until tex_release() has recorded a "last use" event on the
// launching stream (one event per stream that used the entry); eviction takes the least
// recently used unpinned entry, waits for all of its events (the last kernels reading
// through it) and destroys the object, so a texture is never destroyed under a running
// kernel.

struct TexEntry {
  int dev;
  const void* ptr;
  int64_t n;
  cudaTextureObject_t tex;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;  // last launch reading tex, per stream
  uint64_t tick;  // LRU clock
  int pins;       // lookups whose launch has not been recorded yet
};
std::mutex g_tex_mu;
std::vector<TexEntry> g_tex;
uint64_t g_tex_clock = 0;
constexpr size_t TEX_CACHE_MAX = 64;

// returns 0 (use LDG) when the array cannot be a texture; otherwise pinned until tex_release
cudaTextureObject_t weights_texture(const float* w, int64_t n) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(g_tex_mu);
  for (auto& e : g_tex)
    if (e.dev == dev && e.ptr == (const void*)w && e.n == n) {
      e.tick = ++g_tex_clock;
      ++e.pins;
      return e.tex;
    }
  int maxw = 0, align = 0;
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DLinearWidth, dev);
  cudaDeviceGetAttribute(&align, cudaDevAttrTextureAlignment, dev);
  if (n > (int64_t)maxw || (align > 0 && ((uintptr_t)w % (uintptr_t)align) != 0)) return 0;
  size_t slot = g_tex.size();
  if (g_tex.size() >= TEX_CACHE_MAX) {  // evict the least recently used unpinned entry
    uint64_t best = UINT64_MAX;
    for (size_t k = 0; k < g_tex.size(); ++k)
      if (g_tex[k].pins == 0 && g_tex[k].tick < best) { best = g_tex[k].tick; slot = k; }
    if (slot == g_tex.size()) return 0;  // every entry is mid-launch on some thread
    TexEntry& v = g_tex[slot];
    int cur = dev;
    if (v.dev != dev) cudaSetDevice(v.dev);
    for (auto& u : v.uses) {
      cudaEventSynchronize(u.second);
      cudaEventDestroy(u.second);
    }
    cudaDestroyTextureObject(v.tex);
    if (v.dev != dev) cudaSetDevice(cur);
    g_tex.erase(g_tex.begin() + (std::ptrdiff_t)slot);
    slot = g_tex.size();
  }
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<float*>(w);
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = sizeof(float) * (size_t)n;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  g_tex.push_back({dev, (const void*)w, n, tex, {}, ++g_tex_clock, 1});
  return tex;
}

// after the launches that read through tex are queued on st: record the last use, unpin
void tex_release(cudaTextureObject_t tex, cudaStream_t st) {
  if (!tex) return;
  std::lock_guard<std::mutex> lk(g_tex_mu);
  for (auto& e : g_tex)
    if (e.tex == tex) {
      --e.pins;
      cudaEvent_t ev = nullptr;
      for (auto& u : e.uses)
        if (u.first == st) ev = u.second;
      if (!ev && e.uses.size() >= 16) {  // bound the per-entry stream list: retire the oldest
        cudaEventSynchronize(e.uses.front().second);
        cudaEventDestroy(e.uses.front().second);
        e.uses.erase(e.uses.begin());
      }
      if (!ev) {
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
          cudaGetLastError();
          cudaStreamSynchronize(st);  // no event to order the eviction: finish the launch now
          return;
        }
        e.uses.emplace_back(st, ev);
      }
      cudaEventRecord(ev, st);
      return;
    }
}

template <int RNG, typename WT>
int launch_generic(int kind, GenericArgs ga, cudaStream_t st) {
  const unsigned grid = (unsigned)((ga.p_end - ga.p0 + RS_THREADS - 1) / RS_THREADS);
  if (kind == MGP_KIND_C1) k_generic<RNG, WT, 1><<<grid, RS_THREADS, 0, st>>>(ga);
  else if (kind == MGP_KIND_C2) k_generic<RNG, WT, 2><<<grid, RS_THREADS, 0, st>>>(ga);
  else k_generic<RNG, WT, 3><<<grid, RS_THREADS, 0, st>>>(ga);
  LAUNCH_CHECK("k_generic");
  return 0;
}

// One resampler call over particles [p0, p_end).  Arguments already validated.
struct Plan {
  int kind, dtype, rng;
  bool nz;  // no zero weights (caller asserted MGP_FLAG_NONZERO)
  bool no_stage = false;  // MGP_FLAG_NO_STAGE
  const void* w;
  int64_t n, n_w, n_part;
  int32_t b, warp;
  uint64_t seed;
  std::vector<int64_t> off;  // Megopolis offsets (host)
  int64_t* d_off = nullptr;  // device copy for the generic path
  int32_t* kstate = nullptr;
  void* cum = nullptr;       // inclusive prefix sum (multinomial / systematic)
  bool half = false;         // run_range ranges are lower-half ranges of the half-split kernel
  int64_t hi_shift = 0;      // half-split: upper-half ancestors land at anc[i - hi_shift]
  // fused apply_ancestors (ResampleArgs::rows_*); rows_out already shifted like the anc pointer
  const void* const* rows_peers = nullptr;
  int64_t rows_local = 0;
  int64_t rows_half = 0;
  uint32_t row_words = 0;
  uint32_t* rows_out = nullptr;
  cudaStream_t alloc_st = nullptr;  // stream of plan_alloc's buffers

  Plan() = default;
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  ~Plan() {  // early-return paths: release whatever plan_free did not
    for (void* q : {(void*)d_off, (void*)kstate, cum})
      if (q) cudaFreeAsync(q, alloc_st);
  }
};

// The half-split Megopolis kernel applies: W = 32, N = 2^k >= 256, 4 particles per thread
// (the Philox stream), offsets in one launch.
bool plan_half_ok(const Plan& p) {
  return p.kind == MGP_KIND_MEGOPOLIS && p.warp == 32 && p.rng == MGP_RNG_PHILOX && p.n >= 256 &&
         (p.n & (p.n - 1)) == 0 && p.b <= OFF_CAP;
}

bool is_prefix_kind(int kind) { return kind == MGP_KIND_MULTINOMIAL || kind == MGP_KIND_SYSTEMATIC; }

// np.cumsum(values) in the weights' dtype, bit-exact (mgp_prefix.cuh)
template <typename WT>
int px_cumsum(const WT* w, int64_t n, WT* cum, cudaStream_t st) {
  Scratch sc(st);
  const int64_t nch = (n + PX_CHUNK - 1) / PX_CHUNK, nsup = (nch + PX_SUPER - 1) / PX_SUPER;
  int32_t *e0 = nullptr, *mode = nullptr, *se0 = nullptr, *smode = nullptr, *scnt = nullptr;
  double *csum = nullptr, *est = nullptr;
  Tx *agg = nullptr, *sagg = nullptr;
  WT *carry = nullptr, *scarry = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const double*)nullptr, (double*)nullptr, (int)nch, st));
  CUDA_TRY(sc.alloc(&csum, sizeof(double) * nch));
  CUDA_TRY(sc.alloc(&est, sizeof(double) * nch));
  CUDA_TRY(sc.alloc(&e0, sizeof(int32_t) * nch));

  CUDA_TRY(sc.alloc(&agg, sizeof(Tx) * PX_CAND * nch));

  CUDA_TRY(sc.alloc(&se0, sizeof(int32_t) * nsup));
  CUDA_TRY(sc.alloc(&smode, sizeof(int32_t) * nsup));
  CUDA_TRY(sc.alloc(&sagg, sizeof(Tx) * PX_CAND * nsup));

  // zeroed together: the super-chunk counters and the resolver's per-chunk carry / mode and
  // per-super-chunk carry (k_px_materialize loads them all before it knows which ones the
  // resolver wrote)
  const size_t zbytes = sizeof(WT) * (nch + nsup) + sizeof(int32_t) * (nch + nsup);
  unsigned char* zero = nullptr;
  CUDA_TRY(sc.alloc(&zero, zbytes));
  carry = reinterpret_cast<WT*>(zero);
  scarry = carry + nch;
  mode = reinterpret_cast<int32_t*>(scarry + nsup);
  scnt = mode + nch;
  CUDA_TRY(sc.alloc(&tmp, tmp_bytes + 16));
  // 16-byte vector accesses in the streaming passes when both arrays allow them
  const bool vec = ((uintptr_t)w % 16 == 0) && ((uintptr_t)cum % 16 == 0);
  // k_px_chunk_sum also zeroes `zero` (zbytes is a multiple of 4)
  uint32_t* zw = reinterpret_cast<uint32_t*>(zero);
  const int64_t zwords = (int64_t)(zbytes / 4);
  if (vec) k_px_chunk_sum<WT, true><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, csum, zw, zwords);
  else k_px_chunk_sum<WT, false><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, csum, zw, zwords);
  LAUNCH_CHECK("k_px_chunk_sum");
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, csum, est, (int)nch, st));
#if MGP_PX_PDL
  {  // programmatic dependent of the scan: the weight loads overlap its tail
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t la{};
    la.gridDim = dim3((unsigned)nch);
    la.blockDim = dim3(PX_THREADS);
    la.stream = st;
    la.attrs = at;
    la.numAttrs = 1;
    if (vec)
      CUDA_TRY(cudaLaunchKernelEx(&la, k_px_aggregate<WT, true>, w, n, nch, (const double*)est, scnt, e0, agg, se0, sagg));
    else
      CUDA_TRY(cudaLaunchKernelEx(&la, k_px_aggregate<WT, false>, w, n, nch, (const double*)est, scnt, e0, agg, se0, sagg));
  }
#else
  if (vec) k_px_aggregate<WT, true><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, nch, est, scnt, e0, agg, se0, sagg);
  else k_px_aggregate<WT, false><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, nch, est, scnt, e0, agg, se0, sagg);
  LAUNCH_CHECK("k_px_aggregate");
#endif
  const int64_t stage = px_stage_bytes(nsup);
  if (stage > 0)
    CUDA_TRY(cudaFuncSetAttribute(k_px_resolve<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PX_STAGE_MAX));
#if MGP_PX_PDL
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(1);
  lc.blockDim = dim3(PXR_THREADS);
  lc.dynamicSmemBytes = (size_t)stage;
  lc.stream = st;
  lc.attrs = pdl;
  lc.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&lc, k_px_resolve<WT>, w, n, nch, nsup, (const int32_t*)e0, (const Tx*)agg,
                              (const int32_t*)se0, (const Tx*)sagg, carry, mode, scarry, smode, cum));
  lc.gridDim = dim3((unsigned)nch);
  lc.blockDim = dim3(PX_THREADS);
  lc.dynamicSmemBytes = 0;
  if (vec)
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_px_materialize<WT, true>, w, n, (const int32_t*)e0, (const Tx*)agg,
                                (const WT*)scarry, (const int32_t*)smode, (const WT*)carry, (const int32_t*)mode, cum));
  else
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_px_materialize<WT, false>, w, n, (const int32_t*)e0, (const Tx*)agg,
                                (const WT*)scarry, (const int32_t*)smode, (const WT*)carry, (const int32_t*)mode, cum));
#else
  k_px_resolve<WT><<<1, PXR_THREADS, (size_t)stage, st>>>(w, n, nch, nsup, e0, agg, se0, sagg, carry, mode, scarry,
                                                          smode, cum);
  LAUNCH_CHECK("k_px_resolve");
  if (vec) k_px_materialize<WT, true><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, e0, agg, scarry, smode, carry, mode, cum);
  else k_px_materialize<WT, false><<<(unsigned)nch, PX_THREADS, 0, st>>>(w, n, e0, agg, scarry, smode, carry, mode, cum);
  LAUNCH_CHECK("k_px_materialize");
#endif
  return 0;
}

int px_cumsum_any(const void* w, int dtype, int64_t n, void* cum, cudaStream_t st) {
  return dtype == MGP_F32 ? px_cumsum<float>((const float*)w, n, (float*)cum, st)
                          : px_cumsum<double>((const double*)w, n, (double*)cum, st);
}

// searches over particles [p0, p_end) of a prefix-sum resampler (cum already built)
int px_search(int kind, const void* cum, int dtype, int64_t n, uint64_t seed, int64_t p0, int64_t p_end,
              int64_t* anc, cudaStream_t st) {
  const int64_t cnt = p_end - p0;
  if (cnt <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>((cnt + 255) / 256, 148 * 64);
  if (kind == MGP_KIND_MULTINOMIAL) {
    const uint64_t base = megores_base(seed);
    int64_t K = 1;
    while (K * 2 * PXM_PER_BUCKET <= n) K *= 2;
    Scratch sc(st);
    int32_t* start = nullptr;
    CUDA_TRY(sc.alloc(&start, sizeof(int32_t) * (K + 1)));
    const unsigned kg = (unsigned)std::min<int64_t>((K + 256) / 256, 148 * 16);
    // each kernel a programmatic dependent of the one before (griddepcontrol.wait at its top):
    // the launch latency overlaps the previous kernel's tail (MGP_PX_PDL)
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = MGP_PX_PDL;
    cudaLaunchConfig_t la{};
    la.blockDim = dim3(256);
    la.stream = st;
    la.attrs = at;
    la.numAttrs = 1;
    if (dtype == MGP_F32) {
      la.gridDim = dim3(kg);
      CUDA_TRY(cudaLaunchKernelEx(&la, k_multinomial_buckets<float>, (const float*)cum, n, K, start));
      la.gridDim = dim3(grid);
      CUDA_TRY(cudaLaunchKernelEx(&la, k_multinomial<float>, (const float*)cum, n, base, p0, p_end, K,
                                  (const int32_t*)start, anc));
    } else {
      la.gridDim = dim3(kg);
      CUDA_TRY(cudaLaunchKernelEx(&la, k_multinomial_buckets<double>, (const double*)cum, n, K, start));
      la.gridDim = dim3(grid);
      CUDA_TRY(cudaLaunchKernelEx(&la, k_multinomial<double>, (const double*)cum, n, base, p0, p_end, K,
                                  (const int32_t*)start, anc));
    }
  } else {
    const double u0 = (double)(mix64(megores_key(megores_base(seed), GLOBAL_OFFSET_LANE, 0)) >> 11) * 0x1p-53;
    const unsigned sg = (unsigned)std::min<int64_t>((cnt / PXS_RUN + 256) / 256, 148 * 64);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = MGP_PX_PDL;
    cudaLaunchConfig_t la{};
    la.gridDim = dim3(sg);
    la.blockDim = dim3(256);
    la.stream = st;
    la.attrs = at;
    la.numAttrs = 1;
    if (dtype == MGP_F32) CUDA_TRY(cudaLaunchKernelEx(&la, k_systematic<float>, (const float*)cum, n, u0, p0, p_end, anc));
    else CUDA_TRY(cudaLaunchKernelEx(&la, k_systematic<double>, (const double*)cum, n, u0, p0, p_end, anc));
  }
  return 0;
}

bool plan_uses_w32(const Plan& p) {
  if (is_prefix_kind(p.kind)) return false;
  if (p.kind == MGP_KIND_METROPOLIS) return true;
  return p.warp == 32 && p.n % 32 == 0;
}

int run_range(Plan& p, int64_t p0, int64_t p_end, int64_t* anc, cudaStream_t st) {
  if (p0 >= p_end) return 0;
  if (is_prefix_kind(p.kind)) return px_search(p.kind, p.cum, p.dtype, p.n, p.seed, p0, p_end, anc, st);
  if (!plan_uses_w32(p)) {
    GenericArgs ga{p.w, p.n, (int64_t)p.warp, p.n_w, p.n_part, (int64_t)p.b, p0, p_end, p.seed, megores_base(p.seed),
                   p.d_off, anc};
    if (p.rng == MGP_RNG_MEGORES)
      return p.dtype == MGP_F32 ? launch_generic<RNG_MEGORES, float>(p.kind, ga, st)
                                : launch_generic<RNG_MEGORES, double>(p.kind, ga, st);
    return p.dtype == MGP_F32 ? launch_generic<RNG_PHILOX, float>(p.kind, ga, st)
                              : launch_generic<RNG_PHILOX, double>(p.kind, ga, st);
  }
  ResampleArgs a{};
  a.w = p.w;
  a.n = (uint32_t)p.n;
  a.p0 = (uint32_t)p0;
  a.p_end = (uint32_t)p_end;
  a.n_w = (uint32_t)p.n_w;
  a.n_part = (uint32_t)p.n_part;
  a.seed = p.seed;
  a.base = megores_base(p.seed);
  a.kstate = p.kstate;
  a.anc = anc;
  a.one = 1;
  a.half = p.half ? 1 : 0;
  a.hi_shift = p.hi_shift;
  a.rows_peers = p.rows_peers;
  a.rows_local = p.rows_local;
  a.rows_half = p.rows_half;
  a.row_words = p.row_words;
  a.rows_out = p.rows_out;
  {
    uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
    for (int r = 0; r < 10; ++r) { a.pk0[r] = k0; a.pk1[r] = k1; k0 += PHILOX_W0; k1 += PHILOX_W1; }
  }
  if (p.kind == MGP_KIND_MEGOPOLIS && p.dtype == MGP_F32) a.tex = weights_texture((const float*)p.w, p.n);
  struct TexPin {  // unpin (recording the last use on st) on every return path
    cudaTextureObject_t t;
    cudaStream_t s;
    ~TexPin() { tex_release(t, s); }
  } tex_pin{a.tex, st};
  const int cap = (p.kind == MGP_KIND_MEGOPOLIS) ? OFF_CAP : p.b;  // only Megopolis carries params
  for (int b0 = 0; b0 < p.b; b0 += cap) {
    a.b0 = b0;
    a.cnt = std::min(cap, p.b - b0);
    a.first = (b0 == 0);
    a.last = (b0 + a.cnt >= p.b);
    int rc = 0;
    if (p.kind == MGP_KIND_MEGOPOLIS) {
      static thread_local OffChunk oc;
      for (int t = 0; t < a.cnt; ++t) {
        const uint32_t o = (uint32_t)p.off[b0 + t];
        oc.o[t] = make_uint2(o & ~31u, o & 31u);
      }
      const bool pow2 = is_pow2(p.n) && p.n >= 64;
      if (p.rng == MGP_RNG_MEGORES)
        rc = p.dtype == MGP_F32 ? dispatch_mego_w32<RNG_MEGORES, float>(a, oc, pow2, p.nz, st)
                                : dispatch_mego_w32<RNG_MEGORES, double>(a, oc, pow2, p.nz, st);
      else
        rc = p.dtype == MGP_F32 ? dispatch_mego_w32<RNG_PHILOX, float>(a, oc, pow2, p.nz, st)
                                : dispatch_mego_w32<RNG_PHILOX, double>(a, oc, pow2, p.nz, st);
    } else if (p.kind == MGP_KIND_METROPOLIS) {
      const bool pow2 = is_pow2(p.n) && p.n >= 2;
      a.log2 = ilog2((uint64_t)p.n);
      if (p.rng == MGP_RNG_MEGORES)
        rc = p.dtype == MGP_F32 ? dispatch_metro<RNG_MEGORES, float>(a, pow2, p.nz, st)
                                : dispatch_metro<RNG_MEGORES, double>(a, pow2, p.nz, st);
      else
        rc = p.dtype == MGP_F32 ? dispatch_metro<RNG_PHILOX, float>(a, pow2, p.nz, st)
                                : dispatch_metro<RNG_PHILOX, double>(a, pow2, p.nz, st);
    } else {
      const bool pow2 = is_pow2(p.n_w) && p.n_w >= 2;
      a.log2 = ilog2((uint64_t)p.n_w);
      const bool c2 = p.kind == MGP_KIND_C2;
#define C12_GO(R, T) (c2 ? dispatch_c12<R, T, true>(a, pow2, p.nz, p.no_stage, st) : dispatch_c12<R, T, false>(a, pow2, p.nz, p.no_stage, st))
      if (p.rng == MGP_RNG_MEGORES)
        rc = p.dtype == MGP_F32 ? C12_GO(RNG_MEGORES, float) : C12_GO(RNG_MEGORES, double);
      else
        rc = p.dtype == MGP_F32 ? C12_GO(RNG_PHILOX, float) : C12_GO(RNG_PHILOX, double);
#undef C12_GO
    }
    if (rc) return rc;
  }
  return 0;
}

// Validate + build a plan (no data access).
int make_plan(Plan& p, int kind, const void* w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
              int32_t part_bytes, int strict, int rng, int flags) {
  // the prefix-sum methods take no iteration budget (make_resampler ignores b, M/resample.py:450-454)
  if (is_prefix_kind(kind) && rng != MGP_RNG_MEGORES)
    return set_err(MGP_EUNSUPPORTED, "the prefix-sum resamplers draw from the megores stream only");
  int rc = check_common(dtype, n, is_prefix_kind(kind) ? 1 : b, rng);
  if (rc) return rc;
  p.kind = kind;
  p.w = w;
  p.dtype = dtype;
  p.n = n;
  p.b = b;
  p.seed = seed;
  p.rng = rng;
  p.warp = warp;
  p.n_w = 0;
  p.n_part = 0;
  p.nz = (flags & MGP_FLAG_NONZERO) != 0;
  p.no_stage = (flags & MGP_FLAG_NO_STAGE) != 0;
  if (kind == MGP_KIND_MEGOPOLIS) {
    if ((rc = check_warp(n, warp, strict, "megopolis"))) return rc;
    p.off.resize((size_t)b);
    offsets_host(seed, n, b, rng, p.off.data());
  } else if (kind == MGP_KIND_C1 || kind == MGP_KIND_C2) {
    if ((rc = check_warp(n, warp, strict, kind == MGP_KIND_C1 ? "metropolis_c1" : "metropolis_c2"))) return rc;
    if ((rc = check_partition(n, part_bytes, &p.n_w, &p.n_part))) return rc;
  } else if (kind != MGP_KIND_METROPOLIS && !is_prefix_kind(kind)) {
    return set_err(MGP_EINVAL, "unknown resampler kind %d", kind);
  }
  return 0;
}

int plan_alloc(Plan& p, cudaStream_t st) {
  p.alloc_st = st;
  if (is_prefix_kind(p.kind)) {  // the prefix sum is shared by every particle range
    CUDA_TRY(pool_malloc(&p.cum, (size_t)p.n * (p.dtype == MGP_F32 ? 4 : 8), st));
    return px_cumsum_any(p.w, p.dtype, p.n, p.cum, st);
  }
  if (!plan_uses_w32(p) && p.kind == MGP_KIND_MEGOPOLIS) {
    CUDA_TRY(pool_malloc(&p.d_off, sizeof(int64_t) * p.b, st));
    CUDA_TRY(cudaMemcpyAsync(p.d_off, p.off.data(), sizeof(int64_t) * p.b, cudaMemcpyHostToDevice, st));
  }
  if (plan_uses_w32(p) && p.kind == MGP_KIND_MEGOPOLIS && p.b > OFF_CAP)
    CUDA_TRY(pool_malloc(&p.kstate, sizeof(int32_t) * p.n, st));
  return 0;
}

int plan_free(Plan& p, cudaStream_t st) {
  if (p.d_off) CUDA_TRY(cudaFreeAsync(p.d_off, st));
  if (p.kstate) CUDA_TRY(cudaFreeAsync(p.kstate, st));
  if (p.cum) CUDA_TRY(cudaFreeAsync(p.cum, st));
  p.d_off = nullptr;
  p.kstate = nullptr;
  p.cum = nullptr;
  return 0;
}

#ifndef MGP_HOST_CHUNKS
#define MGP_HOST_CHUNKS 16  // lower/upper chunk pairs of the half-split host path
#endif
#ifndef MGP_BATCH_LAST_CHUNKED
#define MGP_BATCH_LAST_CHUNKED 1
#endif
#ifndef MGP_HOST_TAIL_SPLIT
#define MGP_HOST_TAIL_SPLIT 1
#endif

// Chunk boundaries of the host entry over [0, total): chunks of ceil(total / nchunk) (multiples of
// align), the last one cut into a half and two quarters, so the download still to do after the
// last kernel is a quarter of a chunk's (the downloads of the earlier chunks overlap the kernels
// behind them).  Page-locked outputs only: pinned in/out Megopolis 6.66 -> 6.54 ms (Philox),
// 7.94 -> 7.84 (megores) at 2^24; the staged pageable downloads measured ~1 ms slower with the
// extra pieces (scripts/mb/probe_ts.sh).
static std::vector<int64_t> host_chunk_bounds(int64_t total, int64_t nchunk, int64_t align, bool tail_split) {
  int64_t step = (total + nchunk - 1) / nchunk;
  step = (step + align - 1) / align * align;
  std::vector<int64_t> b{0};
  while (b.back() < total) {
    const int64_t c0 = b.back(), rem = total - c0;
    if (rem > step) {
      b.push_back(c0 + step);
      continue;
    }
    if (MGP_HOST_TAIL_SPLIT && tail_split && nchunk > 1) {
      const int64_t h = rem / 2 / align * align, q = rem / 4 / align * align;
      if (q > 0 && h + q < rem) {
        b.push_back(c0 + h);
        b.push_back(c0 + h + q);
      }
    }
    b.push_back(total);
  }
  return b;
}

// ---------------------------------------------------------------------------
// Pageable host buffers.  A cudaMemcpyAsync from or to pageable memory is staged by the
// driver through its own bounce buffer, one copy at a time and synchronously for D2H.  The
// host entry instead streams pageable buffers through page-locked staging slots of its own:
// host threads copy (and first-touch) the pageable side in parallel while the DMA engine
// moves the previous slot, so the pageable copy overlaps both the transfer and the kernel.

// A small persistent pool of host threads (created on first use) for the host-side work of
// the host-buffer entry: the pageable<->staging memcpys, pre-faulting a pageable output while
// the kernels run, and the host weight validation.  A batch of tasks is awaited through its
// own ticket, so concurrent callers share the pool without waiting for each other.
class HostPool {
 public:
  using Ticket = std::shared_ptr<std::atomic<int>>;
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int threads() const { return nthreads_; }
  // queue tasks; returns the ticket to wait on
  Ticket submit(std::vector<std::function<void()>> tasks) {
    auto left = std::make_shared<std::atomic<int>>((int)tasks.size());
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& t : tasks) q_.push_back({std::move(t), left});
    }
    cv_.notify_all();
    return left;
  }
  void wait(const Ticket& t) {
    if (!t) return;
    for (;;) {  // help with queued work while waiting (the caller is a worker too)
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (t->load() == 0) return;
        if (q_.empty()) {
          done_.wait(lk, [&] { return t->load() == 0 || !q_.empty(); });
          continue;
        }
        j = std::move(q_.front());
        q_.pop_front();
      }
      finish(j);
    }
  }
  // n bytes in parallel pieces of at least 1 MiB
  void copy(void* dst, const void* src, size_t n) {
    const size_t piece = std::max<size_t>(1 << 20, (n + nthreads_ - 1) / nthreads_);
    if (n <= piece) { copy_nt(dst, src, n); return; }
    std::vector<std::function<void()>> tasks;
    for (size_t off = 0; off < n; off += piece) {
      const size_t len = std::min(piece, n - off);
      tasks.push_back([=] { copy_nt((char*)dst + off, (const char*)src + off, len); });
    }
    wait(submit(std::move(tasks)));
  }
  // memcpy with streaming (non-temporal) stores for the 16-byte-aligned body: the staged data is
  // written once and not read back by this thread, so the stores skip the read-for-ownership of
  // every destination line (glibc's memcpy switches to streaming stores only far above the
  // 1 MiB pieces used here)
  static void copy_nt(void* dst, const void* src, size_t n) {
#if MGP_COPY_NT && defined(__x86_64__)
    char* d = (char*)dst;
    const char* s = (const char*)src;
    const size_t head = (16 - ((uintptr_t)d & 15)) & 15;
    if (n < 4096 || head > n) { std::memcpy(d, s, n); return; }
    std::memcpy(d, s, head);
    d += head; s += head; n -= head;
    const size_t body = n & ~(size_t)63;
    for (size_t q = 0; q < body; q += 64) {
      const __m128i a = _mm_loadu_si128((const __m128i*)(s + q)), b = _mm_loadu_si128((const __m128i*)(s + q + 16));
      const __m128i c = _mm_loadu_si128((const __m128i*)(s + q + 32)), e = _mm_loadu_si128((const __m128i*)(s + q + 48));
      _mm_stream_si128((__m128i*)(d + q), a);
      _mm_stream_si128((__m128i*)(d + q + 16), b);
      _mm_stream_si128((__m128i*)(d + q + 32), c);
      _mm_stream_si128((__m128i*)(d + q + 48), e);
    }
    _mm_sfence();
    std::memcpy(d + body, s + body, n - body);
#else
    std::memcpy(dst, src, n);
#endif
  }

 private:
  struct Job {
    std::function<void()> fn;
    Ticket left;
  };
  HostPool() {
    // Half the hardware threads, at most 8.  A pool as wide as the machine (16 workers on the 16
    // vCPUs of the B200 boxes) slows the staged downloads to ~9 GB/s: the drop-in call at 2^24
    // takes 21-27 ms (bimodal) instead of 7.6, even when only 8 of the 16 workers take copy
    // pieces (the rest are woken and compete with the thread driving the copy engine and the
    // driver's threads).  4 workers: 7.3-9.4 ms (scripts/mb/dropin_threads.sh).  The weight
    // validation pass costs 1.4 ms at 8 workers against 0.8 at 16.  MGP_HOST_THREADS overrides.
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)std::max(2u, std::min((hw ? hw : 4u) / 2, 8u));
    if (const char* e = getenv("MGP_HOST_THREADS")) nthreads_ = std::max(1, std::min(64, atoi(e)));
    for (int t = 0; t < nthreads_ - 1; ++t) th_.emplace_back([this] { run(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void finish(Job& j) {
    j.fn();
    if (j.left->fetch_sub(1) == 1) {
      std::lock_guard<std::mutex> lk(mu_);
      done_.notify_all();
    }
  }
  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        j = std::move(q_.front());
        q_.pop_front();
      }
      finish(j);
    }
  }
  int nthreads_ = 4;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::deque<Job> q_;
  bool stop_ = false;
};

// Fault in a pageable output buffer (one byte written per 4 KiB page, in parallel) while the
// device works: the staged downloads then copy into resident pages.  The caller overwrites
// every byte afterwards.
HostPool::Ticket prefault(void* h, size_t n) {
  HostPool& hp = HostPool::get();
  const size_t piece = std::max<size_t>(4 << 20, (n + hp.threads() - 1) / hp.threads());
  std::vector<std::function<void()>> tasks;
  for (size_t off = 0; off < n; off += piece) {
    const size_t len = std::min(piece, n - off);
    tasks.push_back([=] {
      volatile char* c = (volatile char*)h + off;
      for (size_t q = 0; q < len; q += 4096) c[q] = 0;
    });
  }
  return hp.submit(std::move(tasks));
}

constexpr size_t STAGE_SLOT = 8u << 20;  // bytes per page-locked staging slot
constexpr int STAGE_SLOTS = 3;
constexpr size_t STAGE_MIN = 4u << 20;   // smaller pageable buffers go through the driver

// Per-thread, per-device streams and events of the host-buffer path, created once (stream
// and event creation would otherwise cost tens of microseconds per call), plus the staging
// slots for pageable buffers (allocated on first pageable use).
struct HostCtx {
  int dev;
  cudaStream_t st, st2, cp;
  std::vector<cudaEvent_t> ev;
  char* stage = nullptr;                // STAGE_SLOTS x STAGE_SLOT page-locked bytes
  cudaEvent_t slot_ev[STAGE_SLOTS] = {};  // last DMA using each slot
};
thread_local std::vector<HostCtx*> g_host_ctx;

int stage_ready(HostCtx* c) {
  if (c->stage) return 0;
  CUDA_TRY(cudaHostAlloc((void**)&c->stage, STAGE_SLOT * STAGE_SLOTS, cudaHostAllocPortable));
  for (auto& e : c->slot_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return 0;
}

// pageable h_src -> device, through the staging slots on stream st (returns after the last
// slot is queued; the DMA of slot k overlaps the host copy into slot k+1)
// MGP_HOST_TRACE=1: per-call phase times of the staged copies on stderr (probes only)
static bool host_trace() {
  static const bool on = getenv("MGP_HOST_TRACE") != nullptr;
  return on;
}
static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int staged_h2d(HostCtx* c, void* d_dst, const void* h_src, size_t n, cudaStream_t st) {
  if (int rc = stage_ready(c)) return rc;
  const bool tr = host_trace();
  double t_ev = 0, t_cp = 0, t0 = tr ? now_ms() : 0;
  int k = 0;
  for (size_t off = 0; off < n; off += STAGE_SLOT, k = (k + 1) % STAGE_SLOTS) {
    const size_t len = std::min(STAGE_SLOT, n - off);
    char* slot = c->stage + (size_t)k * STAGE_SLOT;
    double ta = tr ? now_ms() : 0;
    CUDA_TRY(cudaEventSynchronize(c->slot_ev[k]));  // the slot's previous DMA has drained
    double tb = tr ? now_ms() : 0;
    HostPool::get().copy(slot, (const char*)h_src + off, len);
    if (tr) { const double tc = now_ms(); t_ev += tb - ta; t_cp += tc - tb; }
    CUDA_TRY(cudaMemcpyAsync((char*)d_dst + off, slot, len, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaEventRecord(c->slot_ev[k], st));
  }
  if (tr) fprintf(stderr, "[mgp trace] staged_h2d %zu B: %.2f ms (slot waits %.2f, host copies %.2f)\n", n, now_ms() - t0, t_ev, t_cp);
  return 0;
}

// device -> pageable h_dst for a list of (dst offset, src offset, bytes) pieces, each queued on
// stream cp after its ready event; the host copy of one slot overlaps the DMA of the next
struct StagePiece {
  size_t dst, src, len;
  cudaEvent_t ready;
};
int staged_d2h(HostCtx* c, void* h_dst, const void* d_src, const std::vector<StagePiece>& pieces, cudaStream_t cp,
               const HostPool::Ticket& faulted) {
  if (int rc = stage_ready(c)) return rc;
  std::vector<StagePiece> segs;  // split into slot-sized segments
  for (const auto& p : pieces)
    for (size_t o = 0; o < p.len; o += STAGE_SLOT)
      segs.push_back({p.dst + o, p.src + o, std::min(STAGE_SLOT, p.len - o), o == 0 ? p.ready : nullptr});
  size_t issued = 0;
  auto issue = [&](size_t q) -> cudaError_t {
    const int k = (int)(q % STAGE_SLOTS);
    if (segs[q].ready) {
      const cudaError_t e = cudaStreamWaitEvent(cp, segs[q].ready, 0);
      if (e != cudaSuccess) return e;
    }
    const cudaError_t e = cudaMemcpyAsync(c->stage + (size_t)k * STAGE_SLOT, (const char*)d_src + segs[q].src,
                                          segs[q].len, cudaMemcpyDeviceToHost, cp);
    if (e != cudaSuccess) return e;
    return cudaEventRecord(c->slot_ev[k], cp);
  };
  const bool tr = host_trace();
  cudaEvent_t td[2] = {};  // trace: DMA span on cp
  if (tr) {
    for (auto& e : td) cudaEventCreate(&e);
    cudaEventRecord(td[0], cp);
  }
  for (; issued < segs.size() && issued < (size_t)STAGE_SLOTS - 1; ++issued) CUDA_TRY(issue(issued));
  double t0 = tr ? now_ms() : 0, t_ev = 0, t_cp = 0, t_first = 0;
  HostPool::get().wait(faulted);  // the output's pages are resident before the first host copy
  const double t_fault = tr ? now_ms() - t0 : 0;
  for (size_t q = 0; q < segs.size(); ++q) {
    if (issued < segs.size()) CUDA_TRY(issue(issued++));  // keep the next slots' DMAs in flight
    const int k = (int)(q % STAGE_SLOTS);
    double ta = tr ? now_ms() : 0;
    CUDA_TRY(cudaEventSynchronize(c->slot_ev[k]));
    double tb = tr ? now_ms() : 0;
    HostPool::get().copy((char*)h_dst + segs[q].dst, c->stage + (size_t)k * STAGE_SLOT, segs[q].len);
    if (tr) { const double tc = now_ms(); t_ev += tb - ta; t_cp += tc - tb; if (q == 0) t_first = tb - t0; }
  }
  if (tr) {
    float dm = 0;
    cudaEventRecord(td[1], cp);
    cudaEventSynchronize(td[1]);
    cudaEventElapsedTime(&dm, td[0], td[1]);
    for (auto& e : td) cudaEventDestroy(e);
    fprintf(stderr, "[mgp trace] staged_d2h %zu segs: %.2f ms (prefault wait %.2f, first slot ready %.2f, slot waits %.2f, host copies %.2f; cp stream span %.2f ms)\n",
            segs.size(), now_ms() - t0, t_fault, t_first, t_ev, t_cp, dm);
  }
  return 0;
}

int host_ctx(HostCtx** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  for (HostCtx* c : g_host_ctx)
    if (c->dev == dev) { *out = c; return 0; }
  HostCtx* c = new HostCtx{dev, nullptr, nullptr, nullptr, {}};
  CUDA_TRY(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->cp, cudaStreamNonBlocking));
  c->ev.resize(2 * MGP_HOST_CHUNKS + 8);  // > chunk events + 1: never re-recorded while awaited
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  g_host_ctx.push_back(c);
  *out = c;
  return 0;
}

// true when the host pointer is page-locked (cudaHostAlloc / cudaHostRegister / torch pin_memory)
bool host_is_pinned(const void* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int resample_device(int kind, const void* w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                    int32_t part_bytes, int strict, int rng, int flags, int64_t* anc, void* stream) {
  Plan p;
  int rc = make_plan(p, kind, w, dtype, n, b, seed, warp, part_bytes, strict, rng, flags);
  if (rc) return rc;
  if (!w || !anc) return set_err(MGP_EINVAL, "null pointer");
  cudaStream_t st = S(stream);
  if ((rc = plan_alloc(p, st))) return rc;
  rc = run_range(p, 0, n, anc, st);
  int rc2 = plan_free(p, st);
  return rc ? rc : rc2;
}

}  // namespace

// ===========================================================================
extern "C" {

int mgp_abi_version(void) { return MGP_ABI_VERSION; }

const char* mgp_last_error(void) { return g_err.c_str(); }

int mgp_check_host_weights(const void* h_w, int dtype, int64_t n, int64_t* counts) {
  if ((!h_w && n > 0) || !counts) return set_err(MGP_EINVAL, "null pointer");
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n < 0) return set_err(MGP_EINVAL, "negative length");
  HostPool& hp = HostPool::get();
  const int64_t piece = std::max<int64_t>(1 << 18, (n + hp.threads() - 1) / hp.threads());
  const int64_t np_ = (n + piece - 1) / piece;
  std::vector<std::array<int64_t, 4>> part((size_t)std::max<int64_t>(np_, 1), std::array<int64_t, 4>{0, 0, 0, 0});
  std::vector<std::function<void()>> tasks;
  for (int64_t q = 0; q < np_; ++q) {
    tasks.push_back([=, &part] {
      const int64_t lo = q * piece, hi = std::min(n, lo + piece);
      int64_t nf = 0, ng = 0, nz = 0;
      if (dtype == MGP_F32) {
        const uint32_t* b = (const uint32_t*)h_w;
        for (int64_t i = lo; i < hi; ++i) {
          const uint32_t v = b[i], mag = v & 0x7FFFFFFFu;
          nf += mag >= 0x7F800000u;                       // inf / nan
          ng += (v >> 31) & (mag != 0) & (mag < 0x7F800000u);  // finite and < 0 (-0.0 is not)
          nz += mag == 0;
        }
      } else {
        const uint64_t* b = (const uint64_t*)h_w;
        for (int64_t i = lo; i < hi; ++i) {
          const uint64_t v = b[i], mag = v & 0x7FFFFFFFFFFFFFFFull;
          nf += mag >= 0x7FF0000000000000ull;
          ng += (v >> 63) & (mag != 0) & (mag < 0x7FF0000000000000ull);
          nz += mag == 0;
        }
      }
      part[(size_t)q] = {nf, ng, nz, (hi - lo) - nf - ng - nz};
    });
  }
  hp.wait(hp.submit(std::move(tasks)));
  for (int k = 0; k < 4; ++k) counts[k] = 0;
  for (const auto& pc : part)
    for (int k = 0; k < 4; ++k) counts[k] += pc[k];
  return 0;
}

int mgp_release_cached_memory(int device) {
  int prev = 0;
  CUDA_TRY(cudaGetDevice(&prev));
  if (device >= 0) CUDA_TRY(cudaSetDevice(device));
  cudaMemPool_t pool;
  cudaError_t e = lib_pool(&pool);
  if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
  if (device >= 0) cudaSetDevice(prev);
  return e == cudaSuccess ? 0 : cuda_err(e, "cudaMemPoolTrimTo");
}

int mgp_weight_stats(const void* d_w, int dtype, int64_t n, mgp_weight_stats_t* d_out, void* stream) {
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  PwOut out{&d_out->sum, &d_out->mean, nullptr, reinterpret_cast<WStats*>(&d_out->max)};
  static_assert(sizeof(WStats) == 6 * 8, "WStats layout");
  if (dtype == MGP_F32) {
    const float* w = (const float*)d_w;
    return pw_reduce<ElemWeight<float>, float, true>(ElemWeight<float>{w}, w, n, out, S(stream));
  }
  const double* w = (const double*)d_w;
  return pw_reduce<ElemWeight<double>, double, true>(ElemWeight<double>{w}, w, n, out, S(stream));
}

int mgp_compute_iterations(double epsilon, double mean_w, double max_w, int32_t* b_out) {  // M/weights.py:114-131
  if (!(0.0 < epsilon && epsilon <= 1.0)) return set_err(MGP_EINVAL, "epsilon must be in (0, 1], got %.17g", epsilon);
  if (mean_w <= 0 || max_w <= 0) return set_err(MGP_EINVAL, "mean_w and max_w must be positive");
  if (mean_w > max_w) return set_err(MGP_EINVAL, "mean_w (%.17g) exceeds max_w (%.17g)", mean_w, max_w);
  const double ratio = mean_w / max_w;
  if (ratio >= 1.0 || epsilon == 1.0) { *b_out = 1; return 0; }
  const double v = std::ceil(std::log(epsilon) / std::log(1.0 - ratio));
  if (!(v < 2147483647.0)) return set_err(MGP_EUNSUPPORTED, "B=%.17g exceeds the int32 range", v);
  *b_out = v < 1.0 ? 1 : (int32_t)v;
  return 0;
}

int mgp_offsets_host(uint64_t seed, int64_t n, int32_t b, int rng, int64_t* h_off) {
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1, got %lld", (long long)n);
  if (b < 0) return set_err(MGP_EINVAL, "B must be >= 0");
  if (rng != MGP_RNG_MEGORES && rng != MGP_RNG_PHILOX) return set_err(MGP_EINVAL, "unknown rng stream %d", rng);
  offsets_host(seed, n, b, rng, h_off);
  return 0;
}

int mgp_offsets(uint64_t seed, int64_t n, int32_t b, int rng, int64_t* d_off, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1, got %lld", (long long)n);
  if (b <= 0) return b == 0 ? 0 : set_err(MGP_EINVAL, "B must be >= 0");
  const unsigned grid = (unsigned)((b + 255) / 256);
  if (rng == MGP_RNG_MEGORES) k_offsets<RNG_MEGORES><<<grid, 256, 0, S(stream)>>>(megores_base(seed), seed, n, b, d_off);
  else if (rng == MGP_RNG_PHILOX) k_offsets<RNG_PHILOX><<<grid, 256, 0, S(stream)>>>(0, seed, n, b, d_off);
  else return set_err(MGP_EINVAL, "unknown rng stream %d", rng);
  LAUNCH_CHECK("k_offsets");
  return 0;
}

int mgp_megopolis(const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp, int strict, int rng,
                  int flags, int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_MEGOPOLIS, d_w, dtype, n, b, seed, warp, 0, strict, rng, flags, d_anc, stream);
}

int mgp_metropolis(const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int rng, int flags,
                   int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_METROPOLIS, d_w, dtype, n, b, seed, 32, 0, 0, rng, flags, d_anc, stream);
}

int mgp_metropolis_c1(const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                      int32_t partition_bytes, int strict, int rng, int flags, int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_C1, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags, d_anc, stream);
}

int mgp_metropolis_c2(const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                      int32_t partition_bytes, int strict, int rng, int flags, int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_C2, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags, d_anc, stream);
}

int mgp_resample_range(int kind, const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                       int32_t partition_bytes, int strict, int rng, int flags, int64_t p0, int64_t p1,
                       int64_t* d_anc_slice, void* stream) {
  Plan p;
  int rc = make_plan(p, kind, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags);
  if (rc) return rc;
  if (!d_w || !d_anc_slice) return set_err(MGP_EINVAL, "null pointer");
  if (p0 < 0 || p1 > n || p0 > p1) return set_err(MGP_EINVAL, "particle range [%lld, %lld) outside [0, %lld)",
                                                  (long long)p0, (long long)p1, (long long)n);
  if (plan_uses_w32(p) && p0 % 32) return set_err(MGP_EINVAL, "p0 must be a multiple of 32, got %lld", (long long)p0);
  cudaStream_t st = S(stream);
  if ((rc = plan_alloc(p, st))) return rc;
  rc = run_range(p, p0, p1, d_anc_slice - p0, st);
  int rc2 = plan_free(p, st);
  return rc ? rc : rc2;
}

int mgp_resample_host(int kind, const void* h_w, int dtype, int64_t n, int32_t b, double epsilon, uint64_t seed,
                      int32_t warp, int32_t partition_bytes, int strict, int rng, int64_t* h_anc, int32_t* b_used,
                      int device) {
  if (!h_w || !h_anc) return set_err(MGP_EINVAL, "null pointer");
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N exceeds 2^31-1");
  struct DeviceGuard {  // the caller's current device is restored on every return
    int prev = -1;
    ~DeviceGuard() {
      if (prev >= 0) cudaSetDevice(prev);
    }
  } guard;
  if (device >= 0) {
    CUDA_TRY(cudaGetDevice(&guard.prev));
    CUDA_TRY(cudaSetDevice(device));
  }
  HostCtx* hc = nullptr;
  if (int rc0 = host_ctx(&hc)) return rc0;
  cudaStream_t st = hc->st, st2 = hc->st2, cp = hc->cp;
  size_t next_ev = 0;
  const size_t wbytes = (size_t)n * (dtype == MGP_F32 ? 4 : 8);
  void* d_w = nullptr;
  int64_t* d_anc = nullptr;
  mgp_weight_stats_t* d_stats = nullptr;
  mgp_weight_stats_t hs{};
  int rc = 0;
  Plan p;
  auto cleanup = [&]() {
    cudaStreamSynchronize(cp);
    cudaStreamSynchronize(st2);
    cudaStreamSynchronize(st);
    if (d_w) cudaFreeAsync(d_w, st);
    if (d_anc) cudaFreeAsync(d_anc, st);
    if (d_stats) cudaFreeAsync(d_stats, st);
    plan_free(p, st);
    cudaStreamSynchronize(st);
  };
  auto new_event = [&]() { return hc->ev[next_ev++ % hc->ev.size()]; };
#define HTRY(x)                 \
  do {                          \
    rc = (x);                   \
    if (rc) { cleanup(); return rc; } \
  } while (0)
#define HCUDA(x)                                        \
  do {                                                  \
    cudaError_t e_ = (x);                               \
    if (e_ != cudaSuccess) { rc = cuda_err(e_, #x); cleanup(); return rc; } \
  } while (0)
  HCUDA(pool_malloc(&d_w, wbytes, st));
  HCUDA(pool_malloc(&d_anc, sizeof(int64_t) * n, st));
  HCUDA(pool_malloc(&d_stats, sizeof(mgp_weight_stats_t), st));
  if (wbytes >= STAGE_MIN && !host_is_pinned(h_w)) HTRY(staged_h2d(hc, d_w, h_w, wbytes, st));
  else HCUDA(cudaMemcpyAsync(d_w, h_w, wbytes, cudaMemcpyHostToDevice, st));
  // a pageable output is faulted in by the host pool while the device validates and resamples
  const bool anc_pinned = host_is_pinned(h_anc);
  HostPool::Ticket faulted;
  if (!anc_pinned && sizeof(int64_t) * (size_t)n >= STAGE_MIN) faulted = prefault(h_anc, sizeof(int64_t) * (size_t)n);
  struct FaultWait {  // never return while pool threads still write into h_anc
    const HostPool::Ticket& t;
    ~FaultWait() { HostPool::get().wait(t); }
  } fault_wait{faulted};
  HTRY(mgp_weight_stats(d_w, dtype, n, d_stats, st));
  HCUDA(cudaMemcpyAsync(&hs, d_stats, sizeof hs, cudaMemcpyDeviceToHost, st));
  HCUDA(cudaStreamSynchronize(st));
  // WeightVector.__post_init__ (M/weights.py:56-59) and _check_weights (M/resample.py:96-100)
  if (hs.n_nonfinite) { rc = set_err(MGP_EINVAL, "weights must be finite"); cleanup(); return rc; }
  if (hs.n_neg) { rc = set_err(MGP_EINVAL, "weights must be non-negative"); cleanup(); return rc; }
  if (hs.n_pos == 0) { rc = set_err(MGP_EINVAL, "all weights are zero"); cleanup(); return rc; }
  if (b <= 0) HTRY(mgp_compute_iterations(epsilon, hs.mean, hs.max, &b));
  if (b_used) *b_used = b;
  const int flags = (hs.n_zero == 0) ? MGP_FLAG_NONZERO : 0;
  HTRY(make_plan(p, kind, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags));
  HTRY(plan_alloc(p, st));
  // Overlap the ancestor download with the remaining compute: particle chunks are
  // independent given (w, offsets, seed); each chunk's D2H waits only on its kernel.
  // A D2H into pageable memory returns only once it has completed, so for a pageable h_anc
  // every chunk kernel is queued first and the downloads follow (each still overlaps the
  // chunks behind it); with pinned memory the copies are queued as the chunks are.
  // Pinned h_anc: each chunk's download is queued behind its kernel as the chunks are launched.
  // Pageable h_anc: the chunks are listed with their ready events and, once every chunk kernel
  // is queued, streamed through the page-locked staging slots (staged_d2h: parallel host
  // copies overlap the next slot's DMA and the remaining kernels); small pageable buffers take
  // the driver's own staging after the launches.
  const bool pinned = anc_pinned;
  std::vector<StagePiece> pend;
  auto d2h = [&](int64_t dst, int64_t src, int64_t cnt, cudaEvent_t ready) -> cudaError_t {
    if (!pinned) {
      pend.push_back({sizeof(int64_t) * (size_t)dst, sizeof(int64_t) * (size_t)src, sizeof(int64_t) * (size_t)cnt, ready});
      return cudaSuccess;
    }
    cudaError_t e = cudaStreamWaitEvent(cp, ready, 0);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(h_anc + dst, d_anc + src, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, cp);
  };
  auto flush_pending = [&]() -> int {
    if (pend.empty()) return 0;
    size_t total = 0;
    for (const auto& q : pend) total += q.len;
    if (total >= STAGE_MIN) return staged_d2h(hc, h_anc, d_anc, pend, cp, faulted);
    for (const auto& q : pend) {
      CUDA_TRY(cudaStreamWaitEvent(cp, q.ready, 0));
      CUDA_TRY(cudaMemcpyAsync((char*)h_anc + q.dst, (const char*)d_anc + q.src, q.len, cudaMemcpyDeviceToHost, cp));
    }
    return 0;
  };
  if (plan_half_ok(p)) {  // half-split kernel: chunk c = lower-half range [c0, c1) + its mirror
    p.half = true;
    const int64_t half = n / 2;
    const int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(MGP_HOST_CHUNKS, n >> 20));
    const std::vector<int64_t> bnd = host_chunk_bounds(half, nchunk, 128, anc_pinned);
    // chunk kernels alternate between two streams so each one's drain overlaps the next
    // one's start (they are independent given the weights and offsets)
    cudaEvent_t ready = new_event();
    HCUDA(cudaEventRecord(ready, st));
    HCUDA(cudaStreamWaitEvent(st2, ready, 0));
    cudaEvent_t tk[3] = {};  // MGP_HOST_TRACE: kernel span (start, last chunk on st, on st2)
    if (host_trace()) {
      for (auto& e : tk) cudaEventCreate(&e);
      cudaEventRecord(tk[0], st);
    }
    int k = 0;
    for (; k + 1 < (int)bnd.size(); ++k) {
      const int64_t c0 = bnd[k], c1 = bnd[k + 1];
      cudaStream_t ks = (k & 1) ? st2 : st;
      HTRY(run_range(p, c0, c1, d_anc, ks));
      cudaEvent_t ev = new_event();
      HCUDA(cudaEventRecord(ev, ks));
      HCUDA(d2h(c0, c0, c1 - c0, ev));
      HCUDA(d2h(half + c0, half + c0, c1 - c0, ev));
    }
    if (tk[0]) { cudaEventRecord(tk[1], st); cudaEventRecord(tk[2], st2); }
    HTRY(flush_pending());
    HCUDA(cudaStreamSynchronize(cp));
    HCUDA(cudaStreamSynchronize(st2));
    HCUDA(cudaStreamSynchronize(st));
    if (tk[0]) {
      float a = 0, b2 = 0;
      cudaEventElapsedTime(&a, tk[0], tk[1]);
      cudaEventElapsedTime(&b2, tk[0], tk[2]);
      fprintf(stderr, "[mgp trace] chunk kernels: %.2f ms (st), %.2f ms (st2) after the upload\n", a, b2);
      for (auto& e : tk) cudaEventDestroy(e);
    }
    cleanup();
    return 0;
  }
  const bool chunkable = !(plan_uses_w32(p) && p.kind == MGP_KIND_MEGOPOLIS && p.b > OFF_CAP);
  // ~16 chunks of >= 2^20 particles: the D2H tail after the last kernel is ~1/16 of the download
  const int64_t nchunk = chunkable ? std::max<int64_t>(1, std::min<int64_t>(16, n >> 20)) : 1;
  const std::vector<int64_t> bnd = host_chunk_bounds(n, nchunk, 256, anc_pinned);
  // as above, the chunk kernels alternate between two streams, so the last partial wave of one
  // chunk overlaps the first wave of the next (one stream: 16 drains, ~1 ms at 2^24 for megores)
  {
    cudaEvent_t ready = new_event();
    HCUDA(cudaEventRecord(ready, st));
    HCUDA(cudaStreamWaitEvent(st2, ready, 0));
  }
  for (int kc = 0; kc + 1 < (int)bnd.size(); ++kc) {
    const int64_t c0 = bnd[kc], c1 = bnd[kc + 1];
    cudaStream_t ks = ((kc & 1) && !is_prefix_kind(p.kind)) ? st2 : st;  // searches: one stream measured faster
    HTRY(run_range(p, c0, c1, d_anc, ks));
    cudaEvent_t ev = new_event();
    HCUDA(cudaEventRecord(ev, ks));
    HCUDA(d2h(c0, c0, c1 - c0, ev));
  }
  HTRY(flush_pending());
  HCUDA(cudaStreamSynchronize(cp));
  HCUDA(cudaStreamSynchronize(st2));
  HCUDA(cudaStreamSynchronize(st));
  cleanup();
#undef HTRY
#undef HCUDA
  return 0;
}

// Independent resamples of `count` host weight vectors, pipelined across two device buffer slots:
// job k's upload and statistics run on st2 while job k-1's kernel runs on st, and job k-1's
// download runs on cp while job k's kernel runs.  The host round trip for B (the reference derives
// it on the host) happens while the previous kernel is still running, so consecutive kernels are
// queued back to back.  Same ancestors as `count` calls of mgp_resample_host.
int mgp_resample_host_batch(int kind, const void* const* h_w, int dtype, int64_t n, int32_t count, int32_t b,
                            double epsilon, const uint64_t* seeds, int32_t warp, int32_t partition_bytes, int strict,
                            int rng, int64_t* const* h_anc, int32_t* b_used, int device) {
  if (count < 0) return set_err(MGP_EINVAL, "count must be non-negative");
  if (count == 0) return 0;
  if (!h_w || !h_anc || !seeds) return set_err(MGP_EINVAL, "null pointer");
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N exceeds 2^31-1");
  for (int32_t k = 0; k < count; ++k)
    if (!h_w[k] || !h_anc[k]) return set_err(MGP_EINVAL, "null pointer (job %d)", (int)k);
  struct DeviceGuard {
    int prev = -1;
    ~DeviceGuard() {
      if (prev >= 0) cudaSetDevice(prev);
    }
  } guard;
  if (device >= 0) {
    CUDA_TRY(cudaGetDevice(&guard.prev));
    CUDA_TRY(cudaSetDevice(device));
  }
  HostCtx* hc = nullptr;
  if (int rc0 = host_ctx(&hc)) return rc0;
  cudaStream_t st = hc->st, st2 = hc->st2, cp = hc->cp;
  const size_t wbytes = (size_t)n * (dtype == MGP_F32 ? 4 : 8);
  void* d_w[2] = {nullptr, nullptr};
  int64_t* d_anc[2] = {nullptr, nullptr};
  mgp_weight_stats_t* d_stats[2] = {nullptr, nullptr};
  cudaEvent_t kern_done[2] = {hc->ev[0], hc->ev[1]}, d2h_done[2] = {hc->ev[2], hc->ev[3]};
  Plan plans[2];
  int rc = 0;
  auto cleanup = [&]() {
    cudaStreamSynchronize(cp);
    cudaStreamSynchronize(st2);
    cudaStreamSynchronize(st);
    for (int q = 0; q < 2; ++q) {
      if (d_w[q]) cudaFreeAsync(d_w[q], st);
      if (d_anc[q]) cudaFreeAsync(d_anc[q], st);
      if (d_stats[q]) cudaFreeAsync(d_stats[q], st);
      plan_free(plans[q], st);
    }
    cudaStreamSynchronize(st);
  };
#define BTRY(x)                           \
  do {                                    \
    rc = (x);                             \
    if (rc) { cleanup(); return rc; }     \
  } while (0)
#define BCUDA(x)                                                              \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) { rc = cuda_err(e_, #x); cleanup(); return rc; }   \
  } while (0)
  for (int q = 0; q < 2 && q < count; ++q) {
    BCUDA(pool_malloc(&d_w[q], wbytes, st));
    BCUDA(pool_malloc(&d_anc[q], sizeof(int64_t) * n, st));
    BCUDA(pool_malloc(&d_stats[q], sizeof(mgp_weight_stats_t), st));
  }
  BCUDA(cudaStreamSynchronize(st));  // the slots exist before st2 / cp use them
  for (int32_t k = 0; k < count; ++k) {
    const int q = k & 1;
    if (k >= 2) {
      BCUDA(cudaStreamWaitEvent(st2, kern_done[q], 0));  // job k-2's kernel has read d_w[q]
      BCUDA(cudaStreamWaitEvent(st, d2h_done[q], 0));    // job k-2's download has read d_anc[q]
      BTRY(plan_free(plans[q], st));
    }
    BCUDA(cudaMemcpyAsync(d_w[q], h_w[k], wbytes, cudaMemcpyHostToDevice, st2));
    BTRY(mgp_weight_stats(d_w[q], dtype, n, d_stats[q], st2));
    mgp_weight_stats_t hs{};
    BCUDA(cudaMemcpyAsync(&hs, d_stats[q], sizeof hs, cudaMemcpyDeviceToHost, st2));
    BCUDA(cudaStreamSynchronize(st2));  // job k's weights are on the device and checked
    if (hs.n_nonfinite) { rc = set_err(MGP_EINVAL, "weights must be finite (job %d)", (int)k); cleanup(); return rc; }
    if (hs.n_neg) { rc = set_err(MGP_EINVAL, "weights must be non-negative (job %d)", (int)k); cleanup(); return rc; }
    if (hs.n_pos == 0) { rc = set_err(MGP_EINVAL, "all weights are zero (job %d)", (int)k); cleanup(); return rc; }
    int32_t bk = b;
    if (bk <= 0) BTRY(mgp_compute_iterations(epsilon, hs.mean, hs.max, &bk));
    if (b_used) b_used[k] = bk;
    const int flags = (hs.n_zero == 0) ? MGP_FLAG_NONZERO : 0;
    BTRY(make_plan(plans[q], kind, d_w[q], dtype, n, bk, seeds[k], warp, partition_bytes, strict, rng, flags));
    BTRY(plan_alloc(plans[q], st));
    Plan& pl = plans[q];
    const bool half_ok = plan_half_ok(pl);
    const bool chunk_ok = !(plan_uses_w32(pl) && pl.kind == MGP_KIND_MEGOPOLIS && pl.b > OFF_CAP);
    if (MGP_BATCH_LAST_CHUNKED && k == count - 1 && count > 1 && (n >> 20) > 1 && (half_ok || chunk_ok)) {
      // The last job has no next kernel to hide its download behind: run it in particle chunks
      // (the single-call host entry's schedule, last chunk split) with each chunk's download
      // queued behind its kernel, so only a fraction of the 8N-byte download follows the last
      // kernel instead of all of it (earlier jobs' downloads overlap the next job's kernel).
      const int64_t nchunk = std::min<int64_t>(MGP_HOST_CHUNKS, n >> 20);
      int e = 4;  // hc->ev[0..3] are kern_done / d2h_done
      if (half_ok) {
        pl.half = true;
        const int64_t half = n / 2;
        const std::vector<int64_t> bnd = host_chunk_bounds(half, nchunk, 128, true);
        for (size_t c = 0; c + 1 < bnd.size(); ++c) {
          const int64_t c0 = bnd[c], c1 = bnd[c + 1];
          BTRY(run_range(pl, c0, c1, d_anc[q], st));
          cudaEvent_t ev = hc->ev[e++];
          BCUDA(cudaEventRecord(ev, st));
          BCUDA(cudaStreamWaitEvent(cp, ev, 0));
          BCUDA(cudaMemcpyAsync(h_anc[k] + c0, d_anc[q] + c0, sizeof(int64_t) * (c1 - c0), cudaMemcpyDeviceToHost, cp));
          BCUDA(cudaMemcpyAsync(h_anc[k] + half + c0, d_anc[q] + half + c0, sizeof(int64_t) * (c1 - c0),
                                cudaMemcpyDeviceToHost, cp));
        }
      } else {
        const std::vector<int64_t> bnd = host_chunk_bounds(n, nchunk, 256, true);
        for (size_t c = 0; c + 1 < bnd.size(); ++c) {
          const int64_t c0 = bnd[c], c1 = bnd[c + 1];
          BTRY(run_range(pl, c0, c1, d_anc[q], st));
          cudaEvent_t ev = hc->ev[e++];
          BCUDA(cudaEventRecord(ev, st));
          BCUDA(cudaStreamWaitEvent(cp, ev, 0));
          BCUDA(cudaMemcpyAsync(h_anc[k] + c0, d_anc[q] + c0, sizeof(int64_t) * (c1 - c0), cudaMemcpyDeviceToHost, cp));
        }
      }
      BCUDA(cudaEventRecord(kern_done[q], st));
      BCUDA(cudaEventRecord(d2h_done[q], cp));
      continue;
    }
    BTRY(run_range(pl, 0, n, d_anc[q], st));
    BCUDA(cudaEventRecord(kern_done[q], st));
    BCUDA(cudaStreamWaitEvent(cp, kern_done[q], 0));
    BCUDA(cudaMemcpyAsync(h_anc[k], d_anc[q], sizeof(int64_t) * n, cudaMemcpyDeviceToHost, cp));
    BCUDA(cudaEventRecord(d2h_done[q], cp));
  }
  BCUDA(cudaStreamSynchronize(cp));
  BCUDA(cudaStreamSynchronize(st));
  cleanup();
#undef BTRY
#undef BCUDA
  return 0;
}

#ifndef MGP_OFFSPRING_I32_MIN
#define MGP_OFFSPRING_I32_MIN (1ll << 20)
#endif

// measurement switch (mgp_debug_offspring_mode): 0 = queued (default), 1 = the round-1 int32 atomic
// histogram, 2 = the count-matrix bucketed histogram (round 2 first version), for A/B
static std::atomic<int> g_offspring_mode{0};

int mgp_offspring(const int64_t* d_anc, int64_t n_anc, int64_t n, int64_t* d_counts, int32_t* d_bad, void* stream) {
  if (n < 0 || n_anc < 0) return set_err(MGP_EINVAL, "negative size");
  cudaStream_t st = S(stream);
  // Large histograms: bucketed (no per-particle global atomics; mgp_kernels.cuh k_offb_*)
  const int64_t K = (n + OFFB_BINS - 1) / OFFB_BINS;
  const int64_t tiles = (n_anc + OFFB_TILE - 1) / OFFB_TILE;
  const int mode = g_offspring_mode.load();
  const bool queued = n >= MGP_OFFSPRING_I32_MIN && K <= OFFB_KMAX && n_anc > 0 && n_anc <= MAX_N && mode == 0 &&
                      (((uintptr_t)d_anc) & 15) == 0 && K * (2 * ((n_anc + K - 1) / K) + 1032) < (1ll << 31);
  if (d_bad && !(queued && MGP_OFFQ_PDL)) CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
  Scratch sc(st);
  int32_t* bad = d_bad;
  if (!bad && n_anc) CUDA_TRY(sc.alloc(&bad, sizeof(int32_t)));
  const unsigned grid = (unsigned)((n_anc + 255) / 256);
  // Large histograms: queued (mgp_kernels.cuh k_offq_*): one read of the ancestors, no count pass
  if (queued) {
    constexpr int THR = MGP_OFFQ_THR, PER = MGP_OFFQ_PER;
    constexpr int64_t TILE = (int64_t)PER * THR;
    const bool small_k = 20 * K + 16 + 4 * TILE <= 200 * 1024;  // shared memory per CTA, else half tiles
    const int64_t tile = small_k ? TILE : TILE / 2;
    const int64_t qt = (n_anc + tile - 1) / tile;
    const int64_t avg = (n_anc + K - 1) / K;
    const uint32_t cap = (uint32_t)(((2 * avg + 1024) + 7) & ~7ll);  // queue capacity (uint16 entries)
    uint32_t *ctr = nullptr, *ovf = nullptr;  // ctr: K queue cursors, then the overflow length
    uint16_t* queue = nullptr;
    CUDA_TRY(sc.alloc(&ctr, sizeof(uint32_t) * (K + 1)));
    CUDA_TRY(sc.alloc(&ovf, sizeof(uint32_t) * n_anc));
    CUDA_TRY(sc.alloc(&queue, sizeof(uint16_t) * (size_t)K * cap));
    const size_t ssm = 20 * K + 16 + 4 * tile;
    const size_t hsm = sizeof(uint32_t) * OFFB_BINS;
    CUDA_TRY(cudaFuncSetAttribute(k_offq_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
#if MGP_OFFQ_PDL
    // k_offq_zero (cursors, overflow length, the caller's flag), then each kernel launched as a
    // programmatic dependent of the one before: the scatter's tile loads overlap the zeroing and
    // the launch gaps disappear (mgp_kernels.cuh, MGP_OFFQ_PDL)
    k_offq_zero<<<1, 1024, 0, st>>>(ctr, (int)K + 1, d_bad);
    LAUNCH_CHECK("k_offq_zero");
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)qt);
    lc.blockDim = dim3(THR);
    lc.dynamicSmemBytes = ssm;
    lc.stream = st;
    lc.attrs = pdl;
    lc.numAttrs = 1;
    if (small_k) {
      CUDA_TRY(cudaFuncSetAttribute(k_offq_scatter<THR, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      CUDA_TRY(cudaLaunchKernelEx(&lc, k_offq_scatter<THR, PER>, d_anc, n_anc, n, (int)K, cap, ctr, queue, ctr + K, ovf, bad));
    } else {
      CUDA_TRY(cudaFuncSetAttribute(k_offq_scatter<THR, PER / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      CUDA_TRY(cudaLaunchKernelEx(&lc, k_offq_scatter<THR, PER / 2>, d_anc, n_anc, n, (int)K, cap, ctr, queue, ctr + K, ovf,
                                  bad));
    }
    lc.gridDim = dim3((unsigned)K);
    lc.blockDim = dim3(512);
    lc.dynamicSmemBytes = hsm;
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_offq_hist, (const uint16_t*)queue, cap, (const uint32_t*)ctr, n, d_counts));
    lc.gridDim = dim3(148 * 2);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = 0;
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_offq_overflow, (const uint32_t*)ovf, (const uint32_t*)(ctr + K), d_counts));
#else
    CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(uint32_t) * (K + 1), st));
    if (small_k) {
      CUDA_TRY(cudaFuncSetAttribute(k_offq_scatter<THR, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      k_offq_scatter<THR, PER><<<(unsigned)qt, THR, ssm, st>>>(d_anc, n_anc, n, (int)K, cap, ctr, queue, ctr + K, ovf, bad);
    } else {
      CUDA_TRY(cudaFuncSetAttribute(k_offq_scatter<THR, PER / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      k_offq_scatter<THR, PER / 2><<<(unsigned)qt, THR, ssm, st>>>(d_anc, n_anc, n, (int)K, cap, ctr, queue, ctr + K, ovf,
                                                                   bad);
    }
    LAUNCH_CHECK("k_offq_scatter");
    k_offq_hist<<<(unsigned)K, 512, hsm, st>>>(queue, cap, ctr, n, d_counts);
    LAUNCH_CHECK("k_offq_hist");
    k_offq_overflow<<<148 * 2, 256, 0, st>>>(ovf, ctr + K, d_counts);
    LAUNCH_CHECK("k_offq_overflow");
#endif
    return 0;
  }
  if (n >= MGP_OFFSPRING_I32_MIN && K <= OFFB_KMAX && n_anc > 0 && n_anc <= MAX_N && K * tiles < (1ll << 30) &&
      mode != 1) {
    const int64_t m = K * tiles + 1;  // the bucket-major count matrix plus the total
    uint32_t *mat = nullptr, *off = nullptr;
    uint16_t* runs = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, mat, off, (int)m, st));
    CUDA_TRY(sc.alloc(&mat, sizeof(uint32_t) * m));
    CUDA_TRY(sc.alloc(&off, sizeof(uint32_t) * m));
    CUDA_TRY(sc.alloc(&runs, sizeof(uint16_t) * n_anc));
    CUDA_TRY(sc.alloc(&tmp, tmp_bytes + 16));
    CUDA_TRY(cudaMemsetAsync(mat + (m - 1), 0, sizeof(uint32_t), st));
    k_offb_count<<<(unsigned)tiles, OFFB_THREADS, 0, st>>>(d_anc, n_anc, n, (int)K, tiles, mat, bad);
    LAUNCH_CHECK("k_offb_count");
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, mat, off, (int)m, st));
    const size_t ssm = sizeof(uint32_t) * (3 * K + OFFB_TILE);
    CUDA_TRY(cudaFuncSetAttribute(k_offb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    k_offb_scatter<<<(unsigned)tiles, OFFB_THREADS, ssm, st>>>(d_anc, n_anc, n, (int)K, tiles, mat, off, runs);
    LAUNCH_CHECK("k_offb_scatter");
    const size_t hsm = sizeof(uint32_t) * OFFB_BINS;
    CUDA_TRY(cudaFuncSetAttribute(k_offb_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
    k_offb_hist<<<(unsigned)K, 512, hsm, st>>>(runs, off, tiles, n, d_counts);
    LAUNCH_CHECK("k_offb_hist");
    return 0;
  }
  // Large histograms count in int32 (counts <= n_anc < 2^31): half the footprint of the int64
  // array, so the random-address atomics stay in L2 instead of read-modify-writing DRAM
  // sectors; one streaming pass widens to the ABI's int64.
  if (n >= MGP_OFFSPRING_I32_MIN && n_anc <= MAX_N && (((uintptr_t)d_counts) & 15) == 0) {
    int32_t* c32 = nullptr;
    CUDA_TRY(sc.alloc(&c32, sizeof(int32_t) * n));
    CUDA_TRY(cudaMemsetAsync(c32, 0, sizeof(int32_t) * n, st));
    if (n_anc) {
      k_offspring<int32_t><<<grid, 256, 0, st>>>(d_anc, n_anc, n, c32, bad);
      LAUNCH_CHECK("k_offspring");
    }
    k_widen_counts<<<(unsigned)std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 16), 256, 0, st>>>(c32, n, d_counts);
    LAUNCH_CHECK("k_widen_counts");
    return 0;
  }
  if (n) CUDA_TRY(cudaMemsetAsync(d_counts, 0, sizeof(int64_t) * n, st));
  if (n_anc == 0) return 0;
  k_offspring<int64_t><<<grid, 256, 0, st>>>(d_anc, n_anc, n, d_counts, bad);
  LAUNCH_CHECK("k_offspring");
  return 0;
}

int mgp_expected_offspring(const void* d_w, int dtype, int64_t n, double* d_e, double* d_total, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  cudaStream_t st = S(stream);
  PwOut out{d_total, nullptr, nullptr, nullptr};
  int rc;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dtype == MGP_F32) {
    const float* w = (const float*)d_w;
    if ((rc = pw_reduce<ElemWeight<float>, float, false>(ElemWeight<float>{w}, w, n, out, st))) return rc;
    k_expected<float><<<grid, 256, 0, st>>>(w, n, (double)n, d_total, 0.0, d_e);
  } else if (dtype == MGP_F64) {
    const double* w = (const double*)d_w;
    if ((rc = pw_reduce<ElemWeight<double>, double, false>(ElemWeight<double>{w}, w, n, out, st))) return rc;
    k_expected<double><<<grid, 256, 0, st>>>(w, n, (double)n, d_total, 0.0, d_e);
  } else {
    return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  }
  LAUNCH_CHECK("k_expected");
  return 0;
}

int mgp_expected_offspring_slice(const void* d_w, int dtype, int64_t n_slice, int64_t n_all, double total,
                                 double* d_e, void* stream) {
  if (n_slice < 0 || n_all < 1) return set_err(MGP_EINVAL, "invalid sizes");
  if (!(total > 0)) return set_err(MGP_EINVAL, "total weight must be positive");
  if (n_slice == 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>((n_slice + 255) / 256, 148 * 16);
  if (dtype == MGP_F32) k_expected<float><<<grid, 256, 0, S(stream)>>>((const float*)d_w, n_slice, (double)n_all,
                                                                       nullptr, total, d_e);
  else if (dtype == MGP_F64) k_expected<double><<<grid, 256, 0, S(stream)>>>((const double*)d_w, n_slice,
                                                                             (double)n_all, nullptr, total, d_e);
  else return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  LAUNCH_CHECK("k_expected");
  return 0;
}

int mgp_quality_add(const int64_t* d_counts, const double* d_e, int64_t n, double* d_sum, double* d_sumsq,
                    double* d_se_total, double* d_se_run, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1");
  cudaStream_t st = S(stream);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_quality_accum<int64_t><<<grid, 256, 0, st>>>(d_counts, n, d_sum, d_sumsq);
  LAUNCH_CHECK("k_quality_accum");
  PwOut out{d_se_run, nullptr, d_se_total, nullptr};
  return pw_reduce<ElemSqErr<int64_t>, float, false>(ElemSqErr<int64_t>{d_counts, d_e}, nullptr, n, out, st);
}

int mgp_squared_error(const int64_t* d_counts, const double* d_e, int64_t n, double* d_out, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1");
  PwOut out{d_out, nullptr, nullptr, nullptr};
  return pw_reduce<ElemSqErr<int64_t>, float, false>(ElemSqErr<int64_t>{d_counts, d_e}, nullptr, n, out, S(stream));
}

int mgp_quality_finalize(const double* d_sum, const double* d_sumsq, const double* d_e, int64_t n, int64_t k,
                         double* d_variance, double* d_bias_sq, void* stream) {
  if (k < 2) return set_err(MGP_EINVAL, "need at least 2 runs to estimate variance, got %lld", (long long)k);
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1");
  cudaStream_t st = S(stream);
  int rc;
  PwOut o1{d_variance, nullptr, nullptr, nullptr};
  if ((rc = pw_reduce<ElemVar, float, false>(ElemVar{d_sum, d_sumsq, (double)k}, nullptr, n, o1, st))) return rc;
  PwOut o2{d_bias_sq, nullptr, nullptr, nullptr};
  return pw_reduce<ElemBias, float, false>(ElemBias{d_sum, d_e, (double)k}, nullptr, n, o2, st);
}

int mgp_gather(const void* d_states, int64_t row_bytes, const int64_t* d_anc, int64_t n, void* d_out, void* stream) {
  if (row_bytes < 0 || n < 0) return set_err(MGP_EINVAL, "negative size");
  if (n == 0 || row_bytes == 0) return 0;
  cudaStream_t st = S(stream);
  const uintptr_t al = (uintptr_t)d_states | (uintptr_t)d_out | (uintptr_t)row_bytes;
  const int64_t total_bytes = n * row_bytes;
  auto grid_for = [&](int64_t elems) { return (unsigned)std::min<int64_t>((elems + 255) / 256, 148 * 32); };
  if ((al & 15) == 0) {
    k_gather<uint4><<<grid_for(total_bytes / 16), 256, 0, st>>>((const uint4*)d_states, d_anc, n, row_bytes / 16, (uint4*)d_out);
  } else if ((al & 7) == 0) {
    k_gather<uint2><<<grid_for(total_bytes / 8), 256, 0, st>>>((const uint2*)d_states, d_anc, n, row_bytes / 8, (uint2*)d_out);
  } else if ((al & 3) == 0) {
    k_gather<uint32_t><<<grid_for(total_bytes / 4), 256, 0, st>>>((const uint32_t*)d_states, d_anc, n, row_bytes / 4, (uint32_t*)d_out);
  } else {
    k_gather<uint8_t><<<grid_for(total_bytes), 256, 0, st>>>((const uint8_t*)d_states, d_anc, n, row_bytes, (uint8_t*)d_out);
  }
  LAUNCH_CHECK("k_gather");
  return 0;
}

static int gather_peers(const void* const* peer_states, int npeers, int64_t n_local, int64_t row_bytes,
                        const int64_t* d_anc, int64_t n, void* d_out, void* stream, int64_t rows_half) {
  if (npeers < 1 || npeers > 64) return set_err(MGP_EINVAL, "npeers must be in [1, 64], got %d", npeers);
  if (n_local < 1 || row_bytes < 0 || n < 0) return set_err(MGP_EINVAL, "invalid sizes");
  if (n == 0 || row_bytes == 0) return 0;
  PeerTable pt{};
  uintptr_t al = (uintptr_t)d_out | (uintptr_t)row_bytes;
  for (int r = 0; r < npeers; ++r) {
    if (!peer_states[r]) return set_err(MGP_EINVAL, "null peer pointer %d", r);
    pt.p[r] = peer_states[r];
    al |= (uintptr_t)peer_states[r];
  }
  cudaStream_t st = S(stream);
  const unsigned grid = (unsigned)std::min<int64_t>((n * row_bytes / 4 + 255) / 256 + 1, 148 * 32);
  if ((al & 15) == 0)
    k_gather_peers<uint4><<<grid, 256, 0, st>>>(pt, npeers, n_local, d_anc, n, row_bytes / 16, (uint4*)d_out,
                                                  rows_half);
  else if ((al & 7) == 0)
    k_gather_peers<uint2><<<grid, 256, 0, st>>>(pt, npeers, n_local, d_anc, n, row_bytes / 8, (uint2*)d_out,
                                                  rows_half);
  else if ((al & 3) == 0)
    k_gather_peers<uint32_t><<<grid, 256, 0, st>>>(pt, npeers, n_local, d_anc, n, row_bytes / 4, (uint32_t*)d_out,
                                                  rows_half);
  else
    k_gather_peers<uint8_t><<<grid, 256, 0, st>>>(pt, npeers, n_local, d_anc, n, row_bytes, (uint8_t*)d_out,
                                                  rows_half);
  LAUNCH_CHECK("k_gather_peers");
  return 0;
}

int mgp_gather_peers(const void* const* peer_states, int npeers, int64_t n_local, int64_t row_bytes,
                     const int64_t* d_anc, int64_t n, void* d_out, void* stream) {
  return gather_peers(peer_states, npeers, n_local, row_bytes, d_anc, n, d_out, stream, 0);
}

// ---------------------------------------------------------------------------
// Peer mappings of particle-state arrays (CUDA IPC): one process per GPU exports its
// state array, the others map it (peer access over NVLink enabled lazily), and the
// mapped pointers feed mgp_gather_peers / mgp_resample_gather's owner table.  The
// driver's cuMemGetAddressRange (looked up at run time, so the library does not link
// libcuda) finds the allocation an interior pointer -- e.g. a caching-allocator block --
// belongs to; the handle names that allocation and the offset locates the array in it.

typedef int (*PfnMemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

int mgp_ipc_export(const void* d_ptr, void* handle_out, int64_t* offset_out) {
  if (!d_ptr || !handle_out || !offset_out) return set_err(MGP_EINVAL, "null pointer");
  static PfnMemGetAddressRange range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return set_err(MGP_EUNSUPPORTED, "cuMemGetAddressRange not found");
    range = (PfnMemGetAddressRange)fn;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0)
    return set_err(MGP_EINVAL, "pointer %p is not a device allocation", d_ptr);
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
  return 0;
}

int mgp_ipc_open(const void* handle, int64_t offset, void** d_ptr_out) {
  if (!handle || !d_ptr_out || offset < 0) return set_err(MGP_EINVAL, "invalid argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_ptr_out = (char*)base + offset;
  return 0;
}

int mgp_ipc_close(void* d_ptr, int64_t offset) {
  if (!d_ptr || offset < 0) return set_err(MGP_EINVAL, "invalid argument");
  CUDA_TRY(cudaIpcCloseMemHandle((char*)d_ptr - offset));
  return 0;
}

int mgp_mean(const void* d_x, int dtype, int64_t n, double* d_out, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1");
  PwOut out{nullptr, d_out, nullptr, nullptr};
  if (dtype == MGP_F32) {
    const float* x = (const float*)d_x;
    return pw_reduce<ElemWeight<float>, float, false>(ElemWeight<float>{x}, x, n, out, S(stream));
  }
  if (dtype == MGP_F64) {
    const double* x = (const double*)d_x;
    return pw_reduce<ElemWeight<double>, double, false>(ElemWeight<double>{x}, x, n, out, S(stream));
  }
  return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
}

int mgp_pf_init(int64_t n, uint64_t seed, double sqrt_process_var, double* d_x, void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n_particles must be positive");
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_pf_init<<<grid, 256, 0, S(stream)>>>(n, megores_base(seed), sqrt_process_var, d_x);
  LAUNCH_CHECK("k_pf_init");
  return 0;
}

int mgp_pf_predict_update(const double* d_x, int64_t n, double cos_term, double sqrt_process_var, uint64_t seed,
                          double z, double obs_var, int dtype, double* d_xpred, void* d_w, int32_t* d_any_pos,
                          void* stream) {
  if (n < 1) return set_err(MGP_EINVAL, "n_particles must be positive");
  if (!(obs_var > 0)) return set_err(MGP_EINVAL, "obs_var must be positive");
  const double norm = std::sqrt(2.0 * 3.141592653589793 * obs_var);  // math.sqrt(2.0 * math.pi * obs_var)
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  const uint64_t base = megores_base(seed);
  if (dtype == MGP_F32)
    k_pf_predict_update<float><<<grid, 256, 0, S(stream)>>>(d_x, n, cos_term, sqrt_process_var, base, z, obs_var, norm,
                                                            d_xpred, (float*)d_w, d_any_pos);
  else if (dtype == MGP_F64)
    k_pf_predict_update<double><<<grid, 256, 0, S(stream)>>>(d_x, n, cos_term, sqrt_process_var, base, z, obs_var, norm,
                                                             d_xpred, (double*)d_w, d_any_pos);
  else
    return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  LAUNCH_CHECK("k_pf_predict_update");
  return 0;
}

int mgp_estimate_ratio_stats(const void* d_w, int dtype, int64_t n, int64_t subset, uint64_t seed, double* d_out,
                             void* stream) {
  if (subset < 1 || subset > n) return set_err(MGP_EINVAL, "subset_size must be in [1, %lld], got %lld", (long long)n,
                                               (long long)subset);
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N exceeds 2^31-1");
  cudaStream_t st = S(stream);
  Scratch sc(st);
  mgp_weight_stats_t* ws = nullptr;
  CUDA_TRY(sc.alloc(&ws, sizeof *ws));
  int rc = 0;
  if (subset == n) {  // the full array in natural order (M/weights.py:146-147)
    rc = mgp_weight_stats(d_w, dtype, n, ws, st);
  } else {
    uint64_t *k_in = nullptr, *k_out = nullptr;
    int32_t *i_in = nullptr, *i_out = nullptr;
    double* sub = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    CUDA_TRY(sc.alloc(&k_in, 8 * n));
    CUDA_TRY(sc.alloc(&k_out, 8 * n));
    CUDA_TRY(sc.alloc(&i_in, 4 * n));
    CUDA_TRY(sc.alloc(&i_out, 4 * n));
    CUDA_TRY(sc.alloc(&sub, 8 * subset));
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_ratio_keys<<<grid, 256, 0, st>>>(n, megores_base(seed), k_in, i_in);
    LAUNCH_CHECK("k_ratio_keys");
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, i_in, i_out, (int)n, 0, 53, st));
    CUDA_TRY(sc.alloc(&tmp, tmp_bytes));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, i_in, i_out, (int)n, 0, 53, st));
    const unsigned g2 = (unsigned)std::min<int64_t>((subset + 255) / 256, 148 * 16);
    if (dtype == MGP_F32) k_gather_f64<float><<<g2, 256, 0, st>>>((const float*)d_w, i_out, subset, sub);
    else k_gather_f64<double><<<g2, 256, 0, st>>>((const double*)d_w, i_out, subset, sub);
    LAUNCH_CHECK("k_gather_f64");
    rc = mgp_weight_stats(sub, MGP_F64, subset, ws, st);
  }
  if (!rc) {
    CUDA_TRY(cudaMemcpyAsync(d_out, &ws->mean, sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d_out + 1, &ws->max, sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  return rc;
}

int mgp_comparison_indices(int kind, int64_t n, int32_t b, uint64_t seed, int32_t warp, int32_t partition_bytes,
                           int32_t word_bytes, int64_t* d_out, void* stream) {
  if (kind < MGP_KIND_METROPOLIS || kind > MGP_KIND_MEGOPOLIS)
    return set_err(MGP_EINVAL, "unknown Metropolis-family resampler kind %d", kind);
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1, got %lld", (long long)n);
  if (b < 0) return set_err(MGP_EINVAL, "B must be >= 0, got %d", b);
  if (warp < 1) return set_err(MGP_EINVAL, "warp_size must be positive, got %d", warp);
  int64_t n_w = 0, n_part = 0;
  if (kind == MGP_KIND_C1 || kind == MGP_KIND_C2) {  // PartitionConfig (M/resample.py:78-93)
    if (partition_bytes < 1 || word_bytes < 1 || partition_bytes % word_bytes)
      return set_err(MGP_EINVAL, "partition_bytes must be a positive multiple of word_bytes");
    n_w = partition_bytes / word_bytes;
    if (n % n_w) return set_err(MGP_EINVAL, "N=%lld is not divisible by the partition width %lld", (long long)n,
                                (long long)n_w);
    n_part = n / n_w;
  }
  if (b == 0) return 0;
  cudaStream_t st = S(stream);
  Scratch sc(st);
  int64_t* d_off = nullptr;
  if (kind == MGP_KIND_MEGOPOLIS) {  // megopolis_offsets (M/resample.py:263-265), host like the resampler
    std::vector<int64_t> off((size_t)b);
    offsets_host(seed, n, b, MGP_RNG_MEGORES, off.data());
    CUDA_TRY(sc.alloc(&d_off, sizeof(int64_t) * b));
    CUDA_TRY(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));  // the host vector goes out of scope
  }
  const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)b * n + 255) / 256, 148 * 32);
  k_comparison_indices<<<grid, 256, 0, st>>>(kind, n, b, megores_base(seed), warp, n_w, n_part, d_off, d_out);
  LAUNCH_CHECK("k_comparison_indices");
  return 0;
}

int mgp_traffic_report(const int64_t* d_idx, int64_t rows, int64_t width, int32_t warp, int32_t word_bytes,
                       int32_t segment_bytes, int64_t* d_out, void* stream) {
  if (rows < 0 || width < 0) return set_err(MGP_EINVAL, "negative trace shape");
  if (warp < 1 || warp > 4096) return set_err(MGP_EINVAL, "warp_size must be in [1, 4096], got %d", warp);
  if (word_bytes < 1 || segment_bytes % word_bytes)
    return set_err(MGP_EINVAL, "segment_bytes must be a positive multiple of word_bytes");
  if (width % warp)
    return set_err(MGP_EINVAL, "trace width %lld is not a multiple of the warp size %d", (long long)width, warp);
  cudaStream_t st = S(stream);
  CUDA_TRY(cudaMemsetAsync(d_out, 0, 3 * sizeof(int64_t), st));
  const int64_t groups = rows * (width / warp);
  if (groups == 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>((groups + 255) / 256, 148 * 8);
  k_traffic<<<grid, 256, 0, st>>>(d_idx, groups, warp, word_bytes, segment_bytes, (unsigned long long*)d_out);
  LAUNCH_CHECK("k_traffic");
  return 0;
}

int mgp_gen_gaussian(double y, int64_t n, uint64_t seed, int dtype, void* d_out, void* stream) {
  if (y < 0) return set_err(MGP_EINVAL, "y must be >= 0, got %.17g", y);
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1, got %lld", (long long)n);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  if (dtype == MGP_F32) k_gen_gaussian<float><<<grid, 256, 0, S(stream)>>>(y, n, seed, (float*)d_out);
  else if (dtype == MGP_F64) k_gen_gaussian<double><<<grid, 256, 0, S(stream)>>>(y, n, seed, (double*)d_out);
  else return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  LAUNCH_CHECK("k_gen_gaussian");
  return 0;
}

int mgp_gen_gamma(double alpha, double beta, int64_t n, uint64_t seed, int dtype, void* d_out, void* stream) {
  if (!(alpha > 0) || !(beta > 0))
    return set_err(MGP_EINVAL, "alpha and beta must be > 0, got %.17g, %.17g", alpha, beta);
  if (n < 1) return set_err(MGP_EINVAL, "n must be >= 1, got %lld", (long long)n);
  if (!d_out) return set_err(MGP_EINVAL, "null pointer");
  const double lga = std::lgamma(alpha), scale = 1.0 / beta;  // scipy: ppf * scale, scale = 1 / beta
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  if (dtype == MGP_F32) k_gen_gamma<float><<<grid, 256, 0, S(stream)>>>(alpha, lga, scale, n, seed, (float*)d_out);
  else if (dtype == MGP_F64) k_gen_gamma<double><<<grid, 256, 0, S(stream)>>>(alpha, lga, scale, n, seed, (double*)d_out);
  else return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  LAUNCH_CHECK("k_gen_gamma");
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Philox self-test against curand's device implementation.
namespace {
__global__ void k_philox_selftest(uint64_t key, uint32_t c1, uint32_t c2, uint32_t c3, int64_t n,
                                  unsigned long long* mismatch) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const P4 a = philox4x32_10((uint32_t)i, c1, c2, c3, (uint32_t)key, (uint32_t)(key >> 32));
    const uint4 b = curand_Philox4x32_10(make_uint4((uint32_t)i, c1, c2, c3),
                                         make_uint2((uint32_t)key, (uint32_t)(key >> 32)));
    const int bad = (a.x != b.x) + (a.y != b.y) + (a.z != b.z) + (a.w != b.w);
    if (bad) atomicAdd(mismatch, (unsigned long long)bad);
  }
}
}  // namespace

// Resample and apply the ancestors in the same kernel: the resampled particles' state rows
// are read directly from their owners (peer_rows[owner]: local memory or NVLink-mapped peer
// memory).  layout 0: particles [p0, p1), out_rows[i - p0], owner = anc / rows_local.
// layout 1 (stripes): particles [p0, p1) and N/2 + [p0, p1), outputs [L lower | L upper] like
// mgp_resample_stripes, owner r holding [r*h, (r+1)*h) and N/2 + [r*h, (r+1)*h), h = rows_local/2.
// Fused into the W = 32 kernels' final store; other shapes run mgp_gather_peers afterwards.
extern "C" int mgp_resample_gather(int kind, const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed,
                                   int32_t warp, int32_t partition_bytes, int strict, int rng, int flags, int layout,
                                   int64_t p0, int64_t p1, const void* const* h_peer_rows, int npeers,
                                   int64_t rows_local, int64_t row_bytes, int64_t* d_anc_out, void* d_rows_out,
                                   void* stream) {
  Plan p;
  int rc = make_plan(p, kind, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags);
  if (rc) return rc;
  if (!d_w || !d_anc_out || !h_peer_rows || (!d_rows_out && row_bytes)) return set_err(MGP_EINVAL, "null pointer");
  if (layout != 0 && layout != 1) return set_err(MGP_EINVAL, "layout must be 0 (contiguous) or 1 (stripes)");
  const int64_t half = n / 2, lim = layout ? half : n, L = p1 - p0;
  if (p0 < 0 || p1 > lim || L < 0)
    return set_err(MGP_EINVAL, "particle range [%lld, %lld) outside [0, %lld)", (long long)p0, (long long)p1,
                   (long long)lim);
  if (layout == 1 && (n % 2 || rows_local % 2)) return set_err(MGP_EINVAL, "the stripes layout needs even sizes");
  if (npeers < 1 || npeers > 64 || rows_local < 1 || row_bytes < 0 || rows_local * npeers < n)
    return set_err(MGP_EINVAL, "invalid peer table (npeers=%d, rows_local=%lld, N=%lld)", npeers,
                   (long long)rows_local, (long long)n);
  if (plan_uses_w32(p) && (p0 % 32 || (layout == 1 && half % 32)))
    return set_err(MGP_EINVAL, "p0 (and N/2) must be multiples of 32 for this resampler");
  cudaStream_t st = S(stream);
  uintptr_t al = (uintptr_t)d_rows_out | (uintptr_t)row_bytes;
  for (int r = 0; r < npeers; ++r) {
    if (!h_peer_rows[r]) return set_err(MGP_EINVAL, "null peer pointer %d", r);
    al |= (uintptr_t)h_peer_rows[r];
  }
  const bool fused = plan_uses_w32(p) && row_bytes > 0 && (al & 3) == 0;
  if ((rc = plan_alloc(p, st))) return rc;
  Scratch gsc(st);
  void** d_table = nullptr;
  const int64_t words = row_bytes / 4;
  if (fused) {
    CUDA_TRY(gsc.alloc(&d_table, sizeof(void*) * npeers));
    CUDA_TRY(cudaMemcpyAsync(d_table, h_peer_rows, sizeof(void*) * npeers, cudaMemcpyHostToDevice, st));
    p.rows_peers = (const void* const*)d_table;
    p.rows_local = rows_local;
    p.rows_half = layout ? half : 0;
    p.row_words = (uint32_t)words;
  }
  if (layout == 0) {
    if (fused) p.rows_out = (uint32_t*)d_rows_out - p0 * words;
    rc = run_range(p, p0, p1, d_anc_out - p0, st);
  } else if (plan_half_ok(p) && p0 % 128 == 0 && L % 128 == 0) {
    p.half = true;
    p.hi_shift = half - L;
    if (fused) p.rows_out = (uint32_t*)d_rows_out - p0 * words;
    rc = run_range(p, p0, p1, d_anc_out - p0, st);
  } else {
    if (fused) p.rows_out = (uint32_t*)d_rows_out - p0 * words;
    rc = run_range(p, p0, p1, d_anc_out - p0, st);
    if (fused) p.rows_out = (uint32_t*)d_rows_out + L * words - (half + p0) * words;
    if (!rc) rc = run_range(p, half + p0, half + p1, d_anc_out + L - (half + p0), st);
  }
  if (!rc && !fused && row_bytes > 0) {  // two-kernel route: peer gather with the same owner mapping
    rc = gather_peers(h_peer_rows, npeers, rows_local, row_bytes, d_anc_out, layout ? 2 * L : L, d_rows_out, st,
                      layout ? half : 0);
  }
  int rc2 = plan_free(p, st);
  return rc ? rc : rc2;
}

// Particles [lo0, lo1) and their mirrors [n/2 + lo0, n/2 + lo1) -- the two-stripe ownership
// of the sharded layout (distributed.py, layout="stripes"), which lets every rank run the
// half-split Megopolis kernel.  d_anc_local[0, L) receives the lower stripe, [L, 2L) the upper.
extern "C" int mgp_resample_stripes(int kind, const void* d_w, int dtype, int64_t n, int32_t b, uint64_t seed,
                                    int32_t warp, int32_t partition_bytes, int strict, int rng, int flags,
                                    int64_t lo0, int64_t lo1, int64_t* d_anc_local, void* stream) {
  Plan p;
  int rc = make_plan(p, kind, d_w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags);
  if (rc) return rc;
  if (!d_w || !d_anc_local) return set_err(MGP_EINVAL, "null pointer");
  if (n % 2) return set_err(MGP_EINVAL, "the stripe layout needs an even N, got %lld", (long long)n);
  const int64_t half = n / 2, L = lo1 - lo0;
  if (lo0 < 0 || lo1 > half || L < 0)
    return set_err(MGP_EINVAL, "stripe [%lld, %lld) outside [0, %lld)", (long long)lo0, (long long)lo1, (long long)half);
  if (plan_uses_w32(p) && (lo0 % 32 || half % 32))
    return set_err(MGP_EINVAL, "lo0 and N/2 must be multiples of 32 for this resampler");
  cudaStream_t st = S(stream);
  if ((rc = plan_alloc(p, st))) return rc;
  if (plan_half_ok(p) && lo0 % 128 == 0 && L % 128 == 0) {
    p.half = true;
    p.hi_shift = half - L;
    rc = run_range(p, lo0, lo1, d_anc_local - lo0, st);
  } else {
    rc = run_range(p, lo0, lo1, d_anc_local - lo0, st);
    if (!rc) rc = run_range(p, half + lo0, half + lo1, d_anc_local + L - (half + lo0), st);
  }
  int rc2 = plan_free(p, st);
  return rc ? rc : rc2;
}

// Single-process multi-device resample from host buffers (SURVEY 8b's mgp_megopolis_multi, for C
// hosts without torch.distributed): the weights are replicated to every device (the
// device-to-device copies go peer to peer), device 0 derives B from the numpy-exact stats, and
// device d resamples stripe d of each half (the half-split kernel's pairing; contiguous slices
// when N does not split into stripes) and writes its ancestors straight into h_anc.
extern "C" int mgp_resample_multi(int kind, const void* h_w, int dtype, int64_t n, int32_t b, double epsilon,
                                  uint64_t seed, int32_t warp, int32_t partition_bytes, int strict, int rng,
                                  int ndev, const int* devs, int64_t* h_anc, int32_t* b_used) {
  if (!h_w || !h_anc || !devs) return set_err(MGP_EINVAL, "null pointer");
  if (ndev < 1 || ndev > 64) return set_err(MGP_EINVAL, "ndev must be in [1, 64], got %d", ndev);
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64");
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N exceeds 2^31-1");
  int prev = 0;
  CUDA_TRY(cudaGetDevice(&prev));
  struct Dev {
    int id = 0;
    cudaStream_t st = nullptr;
    void* w = nullptr;
    int64_t* anc = nullptr;
    mgp_weight_stats_t* stats = nullptr;
  };
  std::vector<Dev> dv((size_t)ndev);
  const size_t wbytes = (size_t)n * (dtype == MGP_F32 ? 4 : 8);
  // stripes of h particles per device and half, or contiguous slices of `chunk`
  const int64_t half = n / 2, h = (n % 2 == 0 && half % ndev == 0) ? half / ndev : 0;
  const bool stripes = h > 0 && h % 32 == 0;
  const int64_t chunk = ((n + ndev - 1) / ndev + 31) / 32 * 32;
  int rc = 0;
  cudaEvent_t ready = nullptr;
  auto finish = [&](int code) {
    if (ready) cudaEventDestroy(ready);
    for (auto& d : dv) {
      if (!d.st) continue;
      cudaSetDevice(d.id);
      cudaStreamSynchronize(d.st);
      if (d.w) cudaFreeAsync(d.w, d.st);
      if (d.anc) cudaFreeAsync(d.anc, d.st);
      if (d.stats) cudaFreeAsync(d.stats, d.st);
      cudaStreamSynchronize(d.st);
      cudaStreamDestroy(d.st);
    }
    cudaSetDevice(prev);
    return code;
  };
#define MTRY(x)                                                            \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) return finish(cuda_err(e_, #x));                \
  } while (0)
  for (int d = 0; d < ndev; ++d) {
    Dev& D = dv[(size_t)d];
    D.id = devs[d];
    MTRY(cudaSetDevice(D.id));
    MTRY(cudaStreamCreateWithFlags(&D.st, cudaStreamNonBlocking));
    MTRY(pool_malloc(&D.w, wbytes, D.st));
    MTRY(pool_malloc(&D.anc, sizeof(int64_t) * (stripes ? 2 * h : chunk), D.st));
  }
  // weights: host -> device 0 -> every other device (peer copies)
  MTRY(cudaSetDevice(dv[0].id));
  MTRY(cudaMemcpyAsync(dv[0].w, h_w, wbytes, cudaMemcpyHostToDevice, dv[0].st));
  MTRY(pool_malloc(&dv[0].stats, sizeof(mgp_weight_stats_t), dv[0].st));
  if ((rc = mgp_weight_stats(dv[0].w, dtype, n, dv[0].stats, dv[0].st))) return finish(rc);
  MTRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  MTRY(cudaEventRecord(ready, dv[0].st));
  for (int d = 1; d < ndev; ++d) {
    MTRY(cudaSetDevice(dv[(size_t)d].id));
    MTRY(cudaStreamWaitEvent(dv[(size_t)d].st, ready, 0));
    MTRY(cudaMemcpyPeerAsync(dv[(size_t)d].w, dv[(size_t)d].id, dv[0].w, dv[0].id, wbytes, dv[(size_t)d].st));
  }
  // B rule and validation on the host from device 0's stats (WeightVector / _check_weights)
  mgp_weight_stats_t hs{};
  MTRY(cudaSetDevice(dv[0].id));
  MTRY(cudaMemcpyAsync(&hs, dv[0].stats, sizeof hs, cudaMemcpyDeviceToHost, dv[0].st));
  MTRY(cudaStreamSynchronize(dv[0].st));
  if (hs.n_nonfinite) return finish(set_err(MGP_EINVAL, "weights must be finite"));
  if (hs.n_neg) return finish(set_err(MGP_EINVAL, "weights must be non-negative"));
  if (hs.n_pos == 0) return finish(set_err(MGP_EINVAL, "all weights are zero"));
  if (b <= 0 && (rc = mgp_compute_iterations(epsilon, hs.mean, hs.max, &b))) return finish(rc);
  if (b_used) *b_used = b;
  const int flags = hs.n_zero == 0 ? MGP_FLAG_NONZERO : 0;
  for (int d = 0; d < ndev; ++d) {
    Dev& D = dv[(size_t)d];
    MTRY(cudaSetDevice(D.id));
    if (stripes) {
      const int64_t lo0 = d * h;
      if ((rc = mgp_resample_stripes(kind, D.w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags, lo0,
                                     lo0 + h, D.anc, D.st)))
        return finish(rc);
    } else {
      const int64_t p0 = std::min<int64_t>(n, d * chunk), p1 = std::min<int64_t>(n, p0 + chunk);
      if (p1 <= p0) continue;
      if ((rc = mgp_resample_range(kind, D.w, dtype, n, b, seed, warp, partition_bytes, strict, rng, flags, p0, p1,
                                   D.anc, D.st)))
        return finish(rc);
    }
  }
  // downloads after every device's kernels are queued: a D2H into pageable memory returns
  // only when complete, which would otherwise hold device d+1's launch behind device d
  for (int d = 0; d < ndev; ++d) {
    Dev& D = dv[(size_t)d];
    MTRY(cudaSetDevice(D.id));
    if (stripes) {
      const int64_t lo0 = d * h;
      MTRY(cudaMemcpyAsync(h_anc + lo0, D.anc, sizeof(int64_t) * h, cudaMemcpyDeviceToHost, D.st));
      MTRY(cudaMemcpyAsync(h_anc + half + lo0, D.anc + h, sizeof(int64_t) * h, cudaMemcpyDeviceToHost, D.st));
    } else {
      const int64_t p0 = std::min<int64_t>(n, d * chunk), p1 = std::min<int64_t>(n, p0 + chunk);
      if (p1 <= p0) continue;
      MTRY(cudaMemcpyAsync(h_anc + p0, D.anc, sizeof(int64_t) * (p1 - p0), cudaMemcpyDeviceToHost, D.st));
    }
  }
  for (auto& d : dv) {
    MTRY(cudaSetDevice(d.id));
    MTRY(cudaStreamSynchronize(d.st));
  }
#undef MTRY
  return finish(0);
}

// K resampling runs accumulated into a QualityAccumulator on the device: per seed, the
// resampler, the offspring histogram and QualityAccumulator.add (M/metrics.py:86-93), with no
// host round trip between runs -- the inner loop of the quality grids (M/bench.py:121-126).
extern "C" int mgp_quality_runs(int kind, const void* d_w, int dtype, int64_t n, int32_t b, const uint64_t* h_seeds,
                                int32_t k, int32_t warp, int32_t partition_bytes, int strict, int rng, int flags,
                                const double* d_e, double* d_sum, double* d_sumsq, double* d_se_total, void* stream) {
  if (k < 0 || (k > 0 && !h_seeds)) return set_err(MGP_EINVAL, "invalid seed list");
  if (!d_w || !d_e || !d_sum || !d_sumsq || !d_se_total) return set_err(MGP_EINVAL, "null pointer");
  cudaStream_t st = S(stream);
  Scratch sc(st);
  int64_t *anc = nullptr, *counts = nullptr;
  double* se_run = nullptr;
  CUDA_TRY(sc.alloc(&anc, sizeof(int64_t) * n));
  CUDA_TRY(sc.alloc(&counts, sizeof(int64_t) * n));
  CUDA_TRY(sc.alloc(&se_run, sizeof(double)));
  int rc = 0;
  Plan shared;  // prefix-sum kinds: one prefix sum serves every seed
  const bool prefix = is_prefix_kind(kind);
  if (prefix) {
    rc = make_plan(shared, kind, d_w, dtype, n, b, 0, warp, partition_bytes, strict, rng, flags);
    if (!rc) rc = plan_alloc(shared, st);
  }
  for (int32_t r = 0; r < k && !rc; ++r) {
    if (prefix) {
      shared.seed = h_seeds[r];
      rc = run_range(shared, 0, n, anc, st);
    } else {
      Plan p;
      rc = make_plan(p, kind, d_w, dtype, n, b, h_seeds[r], warp, partition_bytes, strict, rng, flags);
      if (!rc) rc = plan_alloc(p, st);
      if (!rc) rc = run_range(p, 0, n, anc, st);
      int rc2 = plan_free(p, st);
      if (!rc) rc = rc2;
    }
    if (!rc) rc = mgp_offspring(anc, n, n, counts, nullptr, st);
    if (!rc) rc = mgp_quality_add(counts, d_e, n, d_sum, d_sumsq, d_se_total, se_run, st);
  }
  if (prefix) {
    const int rc2 = plan_free(shared, st);
    if (!rc) rc = rc2;
  }
  return rc;
}

extern "C" int mgp_cumsum(const void* d_w, int dtype, int64_t n, void* d_out, void* stream) {
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64, got %d", dtype);
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N=%lld exceeds this build's limit of 2^31-1 particles", (long long)n);
  if (!d_w || !d_out) return set_err(MGP_EINVAL, "null pointer");
  return px_cumsum_any(d_w, dtype, n, d_out, S(stream));
}

extern "C" int mgp_multinomial(const void* d_w, int dtype, int64_t n, uint64_t seed, int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_MULTINOMIAL, d_w, dtype, n, 1, seed, 32, 0, 0, MGP_RNG_MEGORES, 0, d_anc, stream);
}

extern "C" int mgp_systematic(const void* d_w, int dtype, int64_t n, uint64_t seed, int64_t* d_anc, void* stream) {
  return resample_device(MGP_KIND_SYSTEMATIC, d_w, dtype, n, 1, seed, 32, 0, 0, MGP_RNG_MEGORES, 0, d_anc, stream);
}

extern "C" int mgp_systematic_oracle(const void* d_w, int dtype, int64_t n, double u, int64_t* d_anc, void* stream) {
  if (!(u >= 0.0 && u < 1.0)) return set_err(MGP_EINVAL, "u must be in [0, 1), got %.17g", u);
  if (dtype != MGP_F32 && dtype != MGP_F64) return set_err(MGP_EINVAL, "dtype must be MGP_F32 or MGP_F64, got %d", dtype);
  if (n < 1) return set_err(MGP_EINVAL, "weights must be a non-empty 1-d sequence");
  if (n > MAX_N) return set_err(MGP_EUNSUPPORTED, "N=%lld exceeds this build's limit of 2^31-1 particles", (long long)n);
  if (!d_w || !d_anc) return set_err(MGP_EINVAL, "null pointer");
  cudaStream_t st = S(stream);
  Scratch sc(st);
  void* cum = nullptr;
  CUDA_TRY(sc.alloc(&cum, (size_t)n * (dtype == MGP_F32 ? 4 : 8)));
  int rc = px_cumsum_any(d_w, dtype, n, cum, st);
  if (!rc) {
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64);
    if (dtype == MGP_F32) k_systematic_oracle<float><<<grid, 256, 0, st>>>((const float*)cum, n, u, d_anc);
    else k_systematic_oracle<double><<<grid, 256, 0, st>>>((const double*)cum, n, u, d_anc);
    LAUNCH_CHECK("k_systematic_oracle");
  }
  return rc;
}

extern "C" int mgp_philox_selftest(uint64_t key, uint32_t c1, uint32_t c2, uint32_t c3, int64_t n,
                                   int64_t* h_mismatch) {
  Scratch sc(nullptr);
  unsigned long long* d = nullptr;
  CUDA_TRY(sc.alloc(&d, sizeof *d));
  CUDA_TRY(cudaMemset(d, 0, sizeof *d));
  k_philox_selftest<<<148 * 4, 256>>>(key, c1, c2, c3, n, d);
  LAUNCH_CHECK("k_philox_selftest");
  unsigned long long h = 0;
  CUDA_TRY(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
  *h_mismatch = (int64_t)h;
  return 0;
}

extern "C" int mgp_debug_offspring_mode(int mode) {
  if (mode < 0 || mode > 2) return set_err(MGP_EINVAL, "offspring mode must be 0, 1 or 2");
  g_offspring_mode.store(mode);
  return 0;
}

// resolver profile counters of the exact cumsum (non-zero only in a -DMGP_PX_PROF build)
extern "C" int mgp_debug_px_prof(int64_t* h_out16, int reset) {
  CUDA_TRY(cudaMemcpyFromSymbol(h_out16, g_px_prof, sizeof(unsigned long long) * 16));
  if (reset) {
    static const unsigned long long z[16] = {};
    CUDA_TRY(cudaMemcpyToSymbol(g_px_prof, z, sizeof z));
  }
  return 0;
}

extern "C" int mgp_debug_megores_fallbacks(int64_t* h_count, int reset) {
  unsigned long long h = 0;
  CUDA_TRY(cudaMemcpyFromSymbol(&h, g_megores_fallbacks, sizeof h));
  if (reset) {
    const unsigned long long z = 0;
    CUDA_TRY(cudaMemcpyToSymbol(g_megores_fallbacks, &z, sizeof z));
  }
  *h_count = (int64_t)h;
  return 0;
}
