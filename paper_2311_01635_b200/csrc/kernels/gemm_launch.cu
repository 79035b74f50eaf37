// Host-side launchers for the tcgen05 step GEMMs: TMA descriptor encoding
// (operand loads and epilogue stores), tile-size choice, persistent grid
// sizing. No allocation, no sync.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_sm100.cuh"
#include "launch.hpp"

#ifndef RTPB_L2_PROMO
#define RTPB_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

namespace rtpb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

cudaError_t get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? cudaSuccess : cudaErrorNotSupported;
}

// 2-D row-major tensor: `outer` rows of `inner` contiguous elements, row
// stride `ld` elements; box = box_inner x box_outer elements.
int encode_2d(CUtensorMap* m, const void* ptr, bool f32, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  if (get_encode() != cudaSuccess) return set_error(RTPB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t esz = f32 ? 4 : 2;
  if (!ptr) return set_error(RTPB_ERR_DIMENSION, "null operand");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16)
    return set_error(RTPB_ERR_CONFIG,
                     "operand base must be 16-byte aligned and its row stride a multiple of 16 bytes "
                     "(choose dimensions that are multiples of 8)");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        RTPB_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu", int(r),
                  (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld);
    return set_error(RTPB_ERR_CUDA, buf);
  }
  return RTPB_OK;
}

// Epilogue store/reduce map: 32 x 32 boxes, swizzle matching stage_row<>.
int encode_out(CUtensorMap* m, const void* ptr, bool f32, uint64_t cols, uint64_t rows, uint64_t ld) {
  return encode_2d(m, ptr, f32, cols, rows, ld, 32, 32,
                   f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

// Debug timeline buffer (rtpb_debug_trace): each launch takes the next
// gridDim x TRACE_STRIDE block of u64 stamps while space is left.
unsigned long long* g_trace = nullptr;
size_t g_trace_cap = 0, g_trace_next = 0;

unsigned long long* next_trace(unsigned grid) {
  if (!g_trace) return nullptr;
  const size_t need = size_t(grid) * TRACE_STRIDE;
  if (g_trace_next + need > g_trace_cap) return nullptr;
  unsigned long long* p = g_trace + g_trace_next;
  g_trace_next += need;
  return p;
}

int device_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// SMs the next launches of this thread may occupy (set_sm_budget): the
// persistent grid and the tile / split-K choice are sized for them, so two
// GEMMs issued on two streams run side by side instead of queueing.
thread_local int t_sm_budget = 0;
thread_local bool t_pdl = true;
thread_local const unsigned* t_wait_flag = nullptr;
thread_local const unsigned* t_g_flag = nullptr;
thread_local unsigned* t_reset_flags = nullptr;
thread_local unsigned* t_reset_ctr = nullptr;
thread_local int t_reset_count = 0;
// Second K segment of the next launch (gemm_dgrad over two shards): its A
// and B operands, encoded into the launch's second GemmMaps.
struct KSeg {
  bool on = false;
  int kb = 0;
  const void *a, *b;
  uint64_t a_inner, a_outer, a_ld, b_inner, b_outer, b_ld;
};
thread_local KSeg t_kseg;
int sm_count() {
  const int all = device_sms();
  return (t_sm_budget >= 2 && t_sm_budget < all) ? (t_sm_budget & ~1) : all;
}

// Operand: row-major (outer x inner, stride ld); the GEMM reads it MN-major
// (inner = the M/N dimension) or K-major (inner = K) per the kernel config.
struct Op {
  const void* ptr;
  const void* lo;  // TF32X3 low part (same geometry) or nullptr
  uint64_t inner, outer, ld;
};

// Epilogue outputs: c0 (required) and c1 (FWD gelu output, optional).
struct Out {
  const void* ptr;
  bool f32;
  uint64_t cols, rows, ld;
};

template <class Cfg>
int encode_maps(const Op& a, const Op& b, const Out& c0, const Out* c1, GemmMaps& maps) {
  std::memset(&maps, 0, sizeof maps);
  constexpr bool F32 = Cfg::TF32;
  const uint32_t a_box_in = Cfg::A_MN ? Cfg::ATOM_MN : Cfg::BK;
  const uint32_t a_box_out = Cfg::A_MN ? Cfg::BK : Cfg::BM;
  const uint32_t b_box_in = Cfg::B_MN ? Cfg::ATOM_MN : Cfg::BK;
  const uint32_t b_box_out = Cfg::B_MN ? Cfg::BK : Cfg::B_ROWS;  // pair: each CTA stages BN/2 rows
  int rc;
  if ((rc = encode_2d(&maps.a, a.ptr, F32, a.inner, a.outer, a.ld, a_box_in, a_box_out))) return rc;
  if ((rc = encode_2d(&maps.b, b.ptr, F32, b.inner, b.outer, b.ld, b_box_in, b_box_out))) return rc;
  if constexpr (Cfg::TF32) {
    if ((rc = encode_2d(&maps.a_lo, a.lo, F32, a.inner, a.outer, a.ld, a_box_in, a_box_out))) return rc;
    if ((rc = encode_2d(&maps.b_lo, b.lo, F32, b.inner, b.outer, b.ld, b_box_in, b_box_out))) return rc;
  }
  if ((rc = encode_out(&maps.c0, c0.ptr, c0.f32, c0.cols, c0.rows, c0.ld))) return rc;
  const Out& o1 = c1 ? *c1 : c0;  // keep c1 a valid map even when unused
  if ((rc = encode_out(&maps.c1, o1.ptr, o1.f32, o1.cols, o1.rows, o1.ld))) return rc;
  return RTPB_OK;
}

// The kernel's dynamic shared memory opt-in, once per instantiation and
// device. preload_device_kernels sets it for every instantiation up front:
// setting a kernel's attribute may wait for running instances of it, which
// deadlocks when those spin on work the caller has yet to launch.
template <class Cfg>
int set_smem_attr() {
  static unsigned long long done_mask = 0;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard lk(mu);
  if (dev >= 0 && dev < 64 && (done_mask >> dev & 1ull)) return RTPB_OK;
  cudaError_t e = cudaFuncSetAttribute(rtp_gemm_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm)");
  if (dev >= 0 && dev < 64) done_mask |= 1ull << dev;
  return RTPB_OK;
}

// maps2: problem 1 of a scheduled launch (args.sched); slots_override: the
// unit slots (CTA pairs / CTAs) the schedule was built for.
template <class Cfg>
int launch_cfg(const Op& a, const Op& b, const Out& c0, const Out* c1, const GemmArgs& args, cudaStream_t stream,
               const GemmMaps* maps2 = nullptr, int slots_override = 0) {
  GemmMaps maps;
  int rc;
  if ((rc = encode_maps<Cfg>(a, b, c0, c1, maps))) return rc;
  GemmMaps kseg_maps;
  if (t_kseg.on) {
    if (maps2 || args.sched || Cfg::TF32) return set_error(RTPB_ERR_CONFIG, "two K segments: single bf16 problem only");
    const Op a2{t_kseg.a, nullptr, t_kseg.a_inner, t_kseg.a_outer, t_kseg.a_ld};
    const Op b2{t_kseg.b, nullptr, t_kseg.b_inner, t_kseg.b_outer, t_kseg.b_ld};
    if ((rc = encode_maps<Cfg>(a2, b2, c0, c1, kseg_maps))) return rc;
    maps2 = &kseg_maps;
  }
  if ((rc = set_smem_attr<Cfg>())) return rc;  // (normally done by preload_device_kernels)
  int tiles = ((args.M + Cfg::TILE_M - 1) / Cfg::TILE_M) * ((args.N + Cfg::BN - 1) / Cfg::BN) *
              (args.k_splits > 1 ? args.k_splits : 1);  // work units
  if (args.pass_steps && Cfg::EPI == EPI_FWD) tiles *= args.pass_steps;  // flat (step, tile) units
  // Persistent grid: one CTA pair (cluster of 2 on a TPC) per 256-row tile
  // slot, or one CTA per SM. Programmatic stream serialization lets the
  // kernel's prologue run under the previous kernel's tail (griddep_wait()
  // guards every global access).
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = t_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int slots = slots_override > 0 ? slots_override : std::min(tiles, Cfg::PAIR ? sm_count() / 2 : sm_count());
  if constexpr (Cfg::PAIR) {
    cfg.gridDim = dim3(unsigned(2 * slots));
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  } else {
    cfg.gridDim = dim3(unsigned(slots));
  }
  GemmArgs a_ = args;
  if (t_kseg.on) a_.kseg_kb = t_kseg.kb;
  a_.trace = next_trace(cfg.gridDim.x);
  if (!a_.ready_flag) a_.ready_flag = t_wait_flag;  // set_launch_wait_flag()
  if (!a_.g_flag && Cfg::EPI == EPI_WGRAD) a_.g_flag = t_g_flag;  // set_launch_g_flag()
  if (!a_.flag_reset && t_reset_flags) {              // set_launch_flag_reset()
    a_.flag_reset = t_reset_flags;
    a_.flag_reset_ctr = t_reset_ctr;
    a_.flag_reset_count = t_reset_count;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, rtp_gemm_kernel<Cfg>, maps, maps2 ? *maps2 : maps, a_);
  if (e != cudaSuccess) return set_cuda_error(e, "rtp_gemm_kernel launch");
  count_launch();
  return RTPB_OK;
}

// Tile shape: a CTA pair computing 256 x BN (cta_group::2) or one CTA
// computing 128 x BN. Code = BN for single-CTA tiles, 1000 + BN for pairs.
// Choice minimises wave-quantised time: ceil(tiles / slots) * per-tile cost,
// per-tile cost = per-SM work / relative MMA efficiency + fixed overhead
// (relative efficiencies from measured B200 throughput of each shape).
int choose_tile(int M, int N, bool tf32, int mult = 1) {
  struct Cand {
    int code, rows, bn;
    double eff;
  };
  // (eff: measured on B200 at the config (b)/(d) step shapes, tools/tile_sweep.py)
  static const Cand bf16[] = {{1256, 256, 256, 1.00}, {1128, 256, 128, 0.60}, {256, 128, 256, 0.85},
                              {128, 128, 128, 0.62}, {64, 128, 64, 0.32}};
  static const Cand f32[] = {{128, 128, 128, 1.0}, {64, 128, 64, 0.7}};
  const Cand* c = tf32 ? f32 : bf16;
  const int nc = tf32 ? 2 : 5;
  const int sms = sm_count();
  int best = c[0].code;
  double best_cost = -1;
  for (int i = 0; i < nc; ++i) {
    const bool pair = c[i].code > 1000;
    const long tiles = long((M + c[i].rows - 1) / c[i].rows) * ((N + c[i].bn - 1) / c[i].bn) * mult;
    const long slots = pair ? sms / 2 : sms;
    const long waves = (tiles + slots - 1) / slots;
    const double cost = double(waves) * (128.0 * c[i].bn / c[i].eff + 48.0 * 128.0);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = c[i].code;
    }
  }
  return best;
}

constexpr int kEpiWarps = 8;
constexpr int kParMinSplits = 5;  // dW split-K: unordered partials from this many splits

template <int EPI, bool TF32>
int dispatch_tile(int code, const Op& a, const Op& b, const Out& c0, const Out* c1, const GemmArgs& args,
                  cudaStream_t s) {
  constexpr bool AMN = !TF32 && EPI == EPI_WGRAD;
  constexpr bool BMN = !TF32 && EPI != EPI_DGRAD;
  if constexpr (!TF32) {
    if (code == 1256) return launch_cfg<GemmCfg<EPI, 256, false, kEpiWarps, AMN, BMN, false, true>>(a, b, c0, c1, args, s);
    if (code == 1128) return launch_cfg<GemmCfg<EPI, 128, false, kEpiWarps, AMN, BMN, false, true>>(a, b, c0, c1, args, s);
    if (code == 256) return launch_cfg<GemmCfg<EPI, 256, false, kEpiWarps, AMN, BMN>>(a, b, c0, c1, args, s);
  }
  if (code == 64) return launch_cfg<GemmCfg<EPI, 64, TF32, kEpiWarps, AMN, BMN>>(a, b, c0, c1, args, s);
  return launch_cfg<GemmCfg<EPI, 128, TF32, kEpiWarps, AMN, BMN>>(a, b, c0, c1, args, s);
}

// Tile raster: keep one operand L2-resident when it fits (n fastest when all
// of B does: A is streamed once; m fastest when all of A does), else a grouped
// raster over 8 row blocks, whose A and B panels (8 and ~9 of them for a
// machine-wide wave) fit L2 together instead of re-streaming a whole operand
// per wave from HBM.
int raster_mode(int M, int N, int K, int tile_m, int bn, bool f32, bool prefer_m) {
  const double esz = f32 ? 4.0 : 2.0;
  const double a_bytes = double((M + tile_m - 1) / tile_m) * tile_m * K * esz;
  const double b_bytes = double((N + bn - 1) / bn) * bn * K * esz;
  if (prefer_m && a_bytes < 48e6) return 0;
  if (b_bytes < 48e6) return 1;
  if (a_bytes < 48e6) return 0;
  static const int group = [] {  // A/B experiments only (RTPB_RASTER_GROUP)
    const char* e = std::getenv("RTPB_RASTER_GROUP");
    return e ? std::max(2, std::atoi(e)) : 8;
  }();
  return group;
}

bool wave_split_off() {  // A/B: RTPB_NO_WAVE_SPLIT=1
  static const bool off = [] {
    const char* e = std::getenv("RTPB_NO_WAVE_SPLIT");
    return e && std::atoi(e) != 0;
  }();
  return off;
}

// Tile code (and, for dW, the split-K factor written into args.k_splits).
template <int EPI>
int pick_code(bool tf32, GemmArgs& args, int force) {
  int code = force ? force : choose_tile(args.M, args.N, tf32);
  if (tf32 && code > 1000) code -= 1000;  // no pair tiles in the fp32 (3xTF32) mode
  if (tf32 && code == 256) code = 128;
  args.k_splits = 1;
  if (EPI == EPI_WGRAD && !tf32 && args.split_flags) {
    // dW outputs (I x per) are small and K (tokens) long: too few 256x256
    // tiles to occupy every CTA pair. Split K instead of shrinking tiles.
    const int pairs = sm_count() / 2;
    const int tiles = ((args.M + 255) / 256) * ((args.N + 255) / 256);
    const int kb = (args.K + 63) / 64;
    if (!force && tiles < pairs) {
      // The ordered split-K pays one fp32 epilogue per split in sequence
      // (~3 us each for a 256 x 256 pair tile with double-buffered staging,
      // ~1.7 us at 256 x 128) to divide the mainloop (~0.35 us per 64-deep K
      // block at 256 x 256; ~0.27 us at 256 x 128, whose SMs ingest 24 instead
      // of 32 KB per block): take the (width, split) minimising the sum. The
      // narrow tile wins for thin gradient shards (per <= 128: a 256-wide tile
      // would be mostly padding), e.g. config (b) at N = 8.
      int s = 1;
      double best_t = kb * 0.35;
      for (int bn : {256, 128}) {
        const int t_n = ((args.M + 255) / 256) * ((args.N + bn - 1) / bn);
        if (t_n >= pairs) continue;
        const double ck = bn == 256 ? 0.35 : 0.27, ce = bn == 256 ? 3.0 : 1.7;
        const int s_max = std::min(pairs / t_n, std::min(8, kb / 8));
        for (int c = 2; c <= s_max; ++c) {
          const double t = kb * ck / c + ce * c;
          if (t < best_t) {
            best_t = t;
            s = c;
            code = 1000 + bn;
          }
        }
      }
      if (s >= 2) args.k_splits = s;
    } else if (!force && code == 1256 && tiles % pairs != 0 && !wave_split_off()) {
      // Enough tiles for every pair, but the last wave is partial (config (d)
      // at N = 8: 128 pair tiles over 74 pairs = 1.73 waves run as 2). Split
      // K in S ordered parts so the S x tiles units quantise better; the
      // epilogue of a unit overlaps the next unit's mainloop (two TMEM
      // accumulators), the ordered chain's partner is ~tiles units earlier.
      // Time ~ rounds(S) x mainloop / S, +1 exposed epilogue per split.
      const double ck = 0.35, ce = 3.0;
      auto cost = [&](int c) {
        const int rounds = (tiles * c + pairs - 1) / pairs;
        return rounds * std::max(kb * ck / c, ce) + ce * c;
      };
      int s = 1;
      double best_t = cost(1);
      for (int c = 2; c <= 4 && kb / c >= 16; ++c)
        if (cost(c) < 0.95 * best_t) {
          best_t = cost(c);
          s = c;
        }
      if (s >= 2) args.k_splits = s;
    }
  }
  return code;
}

template <int EPI>
int dispatch(bool tf32, const Op& a, const Op& b, const Out& c0, const Out* c1, GemmArgs args, cudaStream_t s,
             int force) {
  const int code = pick_code<EPI>(tf32, args, force);
  const int bn = code % 1000;
  const int num_n = (args.N + bn - 1) / bn;
  (void)num_n;
  const int tile_m = code > 1000 ? 256 : 128;
  // (dW keeps m fastest while its A fits: measured neutral-to-better there)
  args.n_fastest = raster_mode(args.M, args.N, args.K, tile_m, bn, tf32, EPI == EPI_WGRAD);
  return tf32 ? dispatch_tile<EPI, true>(code, a, b, c0, c1, args, s)
              : dispatch_tile<EPI, false>(code, a, b, c0, c1, args, s);
}

// Pass launch (GemmArgs::pass_steps): maps carry buffer 0's B operand and the
// outputs, maps2 buffer 1's B operand (and, DGRAD, the dX output as c0).
template <class Cfg>
int launch_pass(const Op& a, const Op& b0, const Op& b1, const Out& c0, const Out* c1, const Out& d0,
                const Out* d1, const GemmArgs& args, cudaStream_t s, unsigned* done_target) {
  GemmMaps m2;
  int rc;
  if ((rc = encode_maps<Cfg>(a, b1, d0, d1, m2))) return rc;
  const unsigned tiles = unsigned((args.M + Cfg::TILE_M - 1) / Cfg::TILE_M) * unsigned((args.N + Cfg::BN - 1) / Cfg::BN) *
                         unsigned(args.k_splits > 1 ? args.k_splits : 1);  // units per step
  const unsigned target = tiles * unsigned(Cfg::EPI_WARPS * (Cfg::PAIR ? 2 : 1));  // count-ins per step
  // a caller that queued waits for an announced target gets no launch that
  // would count to another one (its waits would never be satisfied)
  if (*done_target && *done_target != target)
    return set_error(RTPB_ERR_STATE, "pass launch: count-in target differs from the announced one");
  *done_target = target;
  return launch_cfg<Cfg>(a, b0, c0, c1, args, s, &m2);
}

template <int EPI>
int dispatch_pass(int code, bool pre_tma, const Op& a, const Op& b0, const Op& b1, const Out& c0, const Out* c1,
                  const Out& d0, const Out* d1, const GemmArgs& args, cudaStream_t s, unsigned* target) {
  constexpr bool BMN = EPI != EPI_DGRAD;
  constexpr bool AMN = EPI == EPI_WGRAD;
  if constexpr (EPI == EPI_DGRAD) {
    if (pre_tma) {
      if (code == 1256)
        return launch_pass<GemmCfg<EPI, 256, false, kEpiWarps, false, false, true, true>>(a, b0, b1, c0, c1, d0, d1,
                                                                                           args, s, target);
      return launch_pass<GemmCfg<EPI, 128, false, kEpiWarps, false, false, true>>(a, b0, b1, c0, c1, d0, d1, args,
                                                                                  s, target);
    }
  }
  if (code == 1256)
    return launch_pass<GemmCfg<EPI, 256, false, kEpiWarps, AMN, BMN, false, true>>(a, b0, b1, c0, c1, d0, d1, args,
                                                                                       s, target);
  if (code == 1128)
    return launch_pass<GemmCfg<EPI, 128, false, kEpiWarps, AMN, BMN, false, true>>(a, b0, b1, c0, c1, d0, d1, args,
                                                                                       s, target);
  if (code == 256)
    return launch_pass<GemmCfg<EPI, 256, false, kEpiWarps, AMN, BMN>>(a, b0, b1, c0, c1, d0, d1, args, s, target);
  if (code == 64)
    return launch_pass<GemmCfg<EPI, 64, false, kEpiWarps, AMN, BMN>>(a, b0, b1, c0, c1, d0, d1, args, s, target);
  return launch_pass<GemmCfg<EPI, 128, false, kEpiWarps, AMN, BMN>>(a, b0, b1, c0, c1, d0, d1, args, s, target);
}

void fill_pass_args(GemmArgs& g, const PassArgs& p) {
  g.pass_steps = p.steps;
  g.pass_pair = p.pair;
  g.pass_buf = p.buf_mask;
  for (int s = 0; s < p.steps; ++s) g.pass_col[s] = p.cols[s];
  g.pass_ready = p.ready;
  g.pass_done = p.done;
  g.flag_reset = p.reset_ctr ? const_cast<unsigned*>(p.ready) : nullptr;
  g.flag_reset_count = p.reset_ctr && p.ready ? p.steps : 0;
  g.flag_reset_ctr = p.reset_ctr;
}

}  // namespace

// The tile code a pass launch of this geometry uses and its count-ins per
// step. The shape is chosen for the pass's units (steps x tiles over the
// slots: one wave-quantisation tail per pass, not per step); the tile shape
// does not change a result's bits (same K order per element; checked by
// tests/test_gpu_pass.py against the per-step launches).
int pass_code(bool dgrad, size_t M, size_t N, bool gelu, int force, int groups) {
  int code = force ? force : choose_tile(int(M), int(N), false, groups);
  if (dgrad && gelu) code = code == 1256 ? 1256 : 128;  // the PRE_TMA shapes (as the last per-step launch)
  return code;
}
unsigned pass_done_target(bool dgrad, size_t M, size_t N, bool gelu, int force, int groups) {
  const int code = pass_code(dgrad, M, N, gelu, force, groups);
  const size_t tm = code > 1000 ? 256 : 128, bn = code % 1000;
  return unsigned(((M + tm - 1) / tm) * ((N + bn - 1) / bn)) * unsigned(kEpiWarps * (code > 1000 ? 2 : 1));
}

int gemm_fwd_pass(const StepFwd& p, const void* w1, size_t y_cols, const PassArgs& pa, cudaStream_t s,
                  unsigned* done_target) {
  // Step s: C[M x per] = X . W(s) with W(s) the I x per block of buffer s.
  Op a{p.x, nullptr, p.I, p.M, p.ldx};
  Op b0{p.w, nullptr, p.per, p.I, p.per}, b1{w1, nullptr, p.per, p.I, p.per};
  GemmArgs g{};
  g.M = int(p.M);
  g.N = int(p.per);
  g.K = int(p.I);
  g.flags = p.flags;
  g.aux = p.bias;
  g.aux2 = p.bias ? static_cast<const char*>(w1) + p.I * p.per * 2 : nullptr;
  fill_pass_args(g, pa);
  // full-width outputs: step s stores at column pass_col[s] + n
  Out y{p.y, false, y_cols, p.M, p.ldy}, act{p.act, false, y_cols, p.M, p.ld_act};
  const bool has_y = (p.flags & EF_STORE_PRE) && p.y;
  const bool has_act = (p.flags & EF_GELU) && p.act;
  const Out& c0 = has_y ? y : act;
  const int code = pass_code(false, p.M, p.per, false, p.force_bn, pa.steps);
  const int bn = code % 1000;
  g.n_fastest = raster_mode(g.M, g.N, g.K, code > 1000 ? 256 : 128, bn, false, false);
  const Out* c1 = has_act ? &act : nullptr;
  return dispatch_pass<EPI_FWD>(code, false, a, b0, b1, c0, c1, c0, c1, g, s, done_target);
}

// dW of every step of a pass into the travelling gradient (GemmArgs
// pass_steps, WGRAD): A = X, B = the whole dY read at the step's column block
// (both MN-major), the per-step split-K of the per-step launches (ordered).
int gemm_wgrad_pass(const StepWgrad& p, size_t dy_cols, bool g_zero, const float* db, const PassArgs& pa,
                    cudaStream_t s, unsigned* done_target) {
  Op a{p.x, nullptr, p.I, p.M, p.ldx};
  Op b{p.dy, nullptr, dy_cols, p.M, p.ldy};
  GemmArgs g{};
  g.M = int(p.I);
  g.N = int(p.per);
  g.K = int(p.M);
  g.flags = g_zero ? EF_FIRST : 0;
  g.split_flags = p.split_flags;
  fill_pass_args(g, pa);
  g.pass_db = db;
  g.pass_gbias = db ? p.g_out + p.I * p.per : nullptr;
  const int code = pick_code<EPI_WGRAD>(false, g, p.force_bn);  // sets g.k_splits
  const int bn = code % 1000;
  g.n_fastest = raster_mode(g.M, g.N, g.K, code > 1000 ? 256 : 128, bn, false, true);
  Out c0{p.g_out, true, p.per, p.I, p.per};
  return dispatch_pass<EPI_WGRAD>(code, false, a, b, b, c0, nullptr, c0, nullptr, g, s, done_target);
}

unsigned wgrad_pass_done_target(size_t M, size_t I, size_t per, int force) {
  GemmArgs g{};
  g.M = int(I);
  g.N = int(per);
  g.K = int(M);
  unsigned dummy = 0;
  g.split_flags = &dummy;
  const int code = pick_code<EPI_WGRAD>(false, g, force);
  const size_t tm = code > 1000 ? 256 : 128, bn = code % 1000;
  return unsigned(((I + tm - 1) / tm) * ((per + bn - 1) / bn) * size_t(g.k_splits > 1 ? g.k_splits : 1)) *
         unsigned(kEpiWarps * (code > 1000 ? 2 : 1));
}

int gemm_dgrad_pass(const StepDgrad& p, const void* w1, size_t dy_cols, const PassArgs& pa, cudaStream_t s,
                    unsigned* done_target) {
  // Step s: acc (+)= dY[:, pass_col[s] :] . W(s)^T; A = the whole dY, K-major,
  // read from column pass_col[s] (K past per multiplies W rows past per: zeros).
  Op a{p.dy, nullptr, dy_cols, p.M, p.ldy};
  Op b0{p.w, nullptr, p.per, p.I, p.per}, b1{w1, nullptr, p.per, p.I, p.per};
  GemmArgs g{};
  g.M = int(p.M);
  g.N = int(p.I);
  g.K = int(p.per);
  g.flags = p.flags & ~(EF_FIRST | EF_LAST);
  g.aux = p.pre;
  g.ld_aux = int64_t(p.ldpre);
  g.acc = p.acc;
  g.ld_acc = int64_t(p.ld_acc);
  fill_pass_args(g, pa);
  Out acc{p.acc, true, p.I, p.M, p.ld_acc}, dx{p.dx, false, p.I, p.M, p.ldx};
  const bool gelu = p.flags & EF_GELU_BWD;
  Out pre{p.pre, false, p.I, p.M, p.ldpre};
  const int code = pass_code(true, p.M, p.I, gelu, p.force_bn, pa.pair ? (pa.steps + 1) / 2 : pa.steps);
  const int bn = code % 1000;
  g.n_fastest = raster_mode(g.M, g.N, g.K, code > 1000 ? 256 : 128, bn, false, false);
  return dispatch_pass<EPI_DGRAD>(code, gelu, a, b0, b1, acc, gelu ? &pre : nullptr, dx, gelu ? &pre : nullptr, g,
                                  s, done_target);
}

// ------------------------------------------------------------------ fused MLP forward (N = 1)
// ffn1 (h -> f, + bias, GELU) and ffn2 (f -> h, + bias) in ONE persistent
// launch on 256 x 256 CTA-pair tiles: problem 0 = ffn1's tiles, problem 1 =
// ffn2's, whose row block mb reads the act rows ffn1's row block mb writes.
// The host assigns units to CTA pairs by greedy list scheduling over a cost
// model (each pair's list in simulated start order, which also makes the
// row-block waits deadlock-free: the earliest-starting blocked unit's
// producers all started earlier and are not blocked), so the two GEMMs share
// one tail instead of paying two wave-quantisation tails.
namespace {
constexpr int kFusedBN = 256;
using FusedFwdCfg = GemmCfg<EPI_FWD, kFusedBN, false, kEpiWarps, false, true, false, true>;

// Cost model of a 256 x 256 CTA-pair tile (us), calibrated on config (b)
// step traces (tools/timeline.py): ~0.36 us per 64-deep K block when TMA-fed
// from L2, plus ~0.85 us per bf16-tile-equivalent written by the epilogue
// (the tile's share of the SM's L2 port), plus a fixed ~0.4 us.
double tile_cost(size_t K, double outputs) { return double((K + 63) / 64) * 0.36 + 0.85 * outputs + 0.4; }

// Two problems on P unit slots. Problem 0: T0 tiles in order (n fastest, n0
// per row block). Problem 1: T1 tiles x S1 K-splits (consecutive units; the
// epilogue of split s follows split s - 1), ready when their row block of
// problem 0 is done (dep 1), when the rows of their K range have been
// published by another launch (dep 2, ext_ready per 256-row block), or at once.
struct TwoProb {
  int T0 = 0, n0 = 0;
  double c0 = 0;
  int T1 = 0, n1 = 0, S1 = 1;
  double c1 = 0;
  int dep = 0;
  const std::vector<double>* ext_ready = nullptr;
  size_t K1 = 0;  // dep 2: problem 1's K (rows of the producing launch)
};

// Greedy list schedule (earliest-free slot takes the next unit). alpha trades
// the two problems: a ready problem-1 unit is taken while its completed
// fraction is <= alpha x problem 0's (alpha < 0: only once problem 0 is
// exhausted). Each slot's list is in simulated start order, which makes the
// kernel's waits deadlock-free. Returns the makespan.
// tail > 0 (dep 1, S1 = 1): the last `tail` problem-1 tiles taken are split
// over K in two units (split code 0 / 1, costing c1_half each; the second's
// epilogue follows the first's), all others run whole (split code 0xFF), so
// the final wave is made of half-length units.
double list_schedule(int P, const TwoProb& q, double alpha, std::vector<int>& sched,
                     std::vector<double>* row_ready_out = nullptr, int tail = 0, double c1_half = 0) {
  std::vector<std::vector<int>> lists(static_cast<size_t>(P));
  std::vector<double> free_at(static_cast<size_t>(P), 0.0);
  const int nm = q.n0 ? (q.T0 + q.n0 - 1) / q.n0 : 1;
  std::vector<double> row_ready(size_t(nm), 0.0);
  std::vector<int> row_left(size_t(nm), q.n0);
  std::vector<int> ready_rows;
  std::vector<double> split_fin(size_t(std::max(q.T1, 1)), 0.0);
  size_t r1 = 0;
  int r1_u = 0, next0 = 0, next1 = 0, taken1 = 0;
  int tiles1 = 0, cur_split = -1;  // tail mode: tiles started, next split of the current tile
  const int U1 = q.T1 * q.S1 + (tail > 0 ? tail : 0);
  double makespan = 0;
  for (int done = 0; done < q.T0 + U1; ++done) {
    int p = 0;
    for (int i = 1; i < P; ++i)
      if (free_at[size_t(i)] < free_at[size_t(p)]) p = i;
    const double tp = free_at[size_t(p)];
    // candidate problem-1 unit and its readiness
    int t1 = -1, sp = 0;
    double rdy = 0.0;
    bool split_tile = false;
    if (q.dep == 1) {
      if (r1 < ready_rows.size()) {
        const int mb = ready_rows[r1];
        t1 = mb * q.n1 + r1_u / q.S1;
        sp = r1_u % q.S1;
        rdy = row_ready[size_t(mb)];
        if (tail > 0) {
          split_tile = tiles1 >= q.T1 - tail;
          sp = split_tile ? (cur_split < 0 ? 0 : cur_split) : 0xFF;
        }
      }
    } else if (next1 < U1) {
      t1 = next1 / q.S1;
      sp = next1 % q.S1;
      if (q.dep == 2 && q.ext_ready && !q.ext_ready->empty()) {
        const size_t rows_per = (q.K1 + size_t(q.S1) - 1) / size_t(q.S1);
        const size_t r_hi = std::min(q.K1, rows_per * size_t(sp + 1));
        const size_t rb = std::min(q.ext_ready->size() - 1, (r_hi ? r_hi - 1 : 0) / 256);
        rdy = (*q.ext_ready)[rb] - 0.9 * q.c1;  // K blocks stream in as rows land
      }
    }
    const double f0 = q.T0 ? double(next0) / q.T0 : 1.0, f1 = U1 ? double(taken1) / U1 : 1.0;
    bool take1 = false;
    if (next0 >= q.T0) take1 = true;
    else if (t1 >= 0 && rdy <= tp && alpha >= 0 && f1 <= alpha * f0) take1 = true;
    double fin;
    if (take1) {
      fin = std::max(tp, rdy) + (split_tile ? c1_half : q.c1);
      if (sp > 0 && sp != 0xFF) fin = std::max(fin, split_fin[size_t(t1)] + 0.6);
      split_fin[size_t(t1)] = fin;
      lists[size_t(p)].push_back((1 << 28) | (sp << 20) | t1);
      ++taken1;
      if (split_tile && sp == 0) {
        cur_split = 1;  // the tile's second half comes next
      } else if (q.dep == 1) {
        cur_split = -1;
        ++tiles1;
        if (++r1_u == q.n1 * q.S1) {
          r1_u = 0;
          ++r1;
        }
      } else {
        ++next1;
      }
    } else {
      const int t = next0++;
      fin = tp + q.c0;
      lists[size_t(p)].push_back(t);
      if (q.n0) {
        const int mb = t / q.n0;
        row_ready[size_t(mb)] = std::max(row_ready[size_t(mb)], fin);
        if (--row_left[size_t(mb)] == 0) ready_rows.push_back(mb);
      }
    }
    free_at[size_t(p)] = fin;
    makespan = std::max(makespan, fin);
  }
  sched.assign(size_t(P) + 1, 0);
  int off = P + 1;
  for (int i = 0; i < P; ++i) {
    sched[size_t(i)] = off;
    off += int(lists[size_t(i)].size());
  }
  sched[size_t(P)] = off;
  for (int i = 0; i < P; ++i) sched.insert(sched.end(), lists[size_t(i)].begin(), lists[size_t(i)].end());
  if (row_ready_out) *row_ready_out = row_ready;
  return makespan;
}

// The same problem scheduled backwards in time (dep 1, S1 = 1): the long
// problem-1 tiles are placed first, then each row block's problem-0 tiles once
// all of that row block's problem-1 tiles are placed; reversing every slot's
// list gives a valid forward schedule whose ragged edge falls on the start,
// among the short problem-0 tiles, instead of on the final long tiles.
double list_schedule_reverse(int P, const TwoProb& q, std::vector<int>& sched, std::vector<double>* row_ready_out) {
  const int nm = q.n0 ? (q.T0 + q.n0 - 1) / q.n0 : 1;
  std::vector<std::vector<std::pair<double, int>>> lists(static_cast<size_t>(P));  // (rev start, code)
  std::vector<double> free_at(static_cast<size_t>(P), 0.0);
  std::vector<double> row_rel(size_t(nm), 0.0);  // rev time all problem-1 tiles of the row are done
  std::vector<int> row_left1(size_t(nm), q.n1);
  std::vector<int> released;  // row blocks in release order
  size_t rel_i = 0;
  int rel_nb = 0, next1 = 0;
  double makespan = 0;
  for (int done = 0; done < q.T0 + q.T1; ++done) {
    int p = 0;
    for (int i = 1; i < P; ++i)
      if (free_at[size_t(i)] < free_at[size_t(p)]) p = i;
    const double tp = free_at[size_t(p)];
    double start, fin;
    if (next1 < q.T1) {
      const int t = next1++, mb = t / q.n1;
      start = tp;
      fin = start + q.c1;
      lists[size_t(p)].push_back({start, (1 << 28) | t});
      row_rel[size_t(mb)] = std::max(row_rel[size_t(mb)], fin);
      if (--row_left1[size_t(mb)] == 0) released.push_back(mb);
    } else {
      // problem-1 tiles all placed: rows are released in order of their release time
      if (rel_i == 0 && rel_nb == 0)
        std::stable_sort(released.begin(), released.end(),
                         [&](int a, int b) { return row_rel[size_t(a)] < row_rel[size_t(b)]; });
      const int mb = released[rel_i];
      const int t = mb * q.n0 + rel_nb;
      if (++rel_nb == q.n0) {
        rel_nb = 0;
        ++rel_i;
      }
      start = std::max(tp, row_rel[size_t(mb)]);
      fin = start + q.c0;
      lists[size_t(p)].push_back({start, t});
    }
    free_at[size_t(p)] = fin;
    makespan = std::max(makespan, fin);
  }
  // real time t' = makespan - t: each slot runs its list backwards
  sched.assign(size_t(P) + 1, 0);
  int off = P + 1;
  for (int i = 0; i < P; ++i) {
    sched[size_t(i)] = off;
    off += int(lists[size_t(i)].size());
  }
  sched[size_t(P)] = off;
  std::vector<double> row_ready(size_t(nm), 0.0);
  for (int i = 0; i < P; ++i)
    for (auto it = lists[size_t(i)].rbegin(); it != lists[size_t(i)].rend(); ++it) {
      sched.push_back(it->second);
      if (!(it->second >> 28) && q.n0) {
        const int mb = it->second / q.n0;
        row_ready[size_t(mb)] = std::max(row_ready[size_t(mb)], makespan - it->first);
      }
    }
  if (row_ready_out) *row_ready_out = row_ready;
  return makespan;
}

const double kAlphas[] = {-1.0, 0.25, 0.5, 0.75, 1.0, 1.25, 1.5, 2.0, 3.0, 1e9};

// Best alpha for a two-problem schedule; returns the makespan.
double best_schedule(int P, const TwoProb& q, std::vector<int>& sched, std::vector<double>* row_ready = nullptr) {
  double best = 1e300;
  if (q.dep == 1 && q.S1 == 1 && !std::getenv("RTPB_NO_REVERSE_SCHED")) {
    std::vector<double> rr;
    best = list_schedule_reverse(P, q, sched, &rr);
    if (row_ready) row_ready->swap(rr);
  }
  for (double al : kAlphas) {
    std::vector<int> s_;
    std::vector<double> rr;
    const double t = list_schedule(P, q, al, s_, &rr);
    if (t < best) {
      best = t;
      sched.swap(s_);
      if (row_ready) row_ready->swap(rr);
    }
  }
  return best;
}
}  // namespace

bool plan_fused_fwd(size_t M, size_t h, size_t f, FusedFwdPlan& plan) {
  const int P = sm_count() / 2;
  const int nm = int((M + 255) / 256), n0 = int((f + kFusedBN - 1) / kFusedBN), n1 = int((h + kFusedBN - 1) / kFusedBN);
  const int T0 = nm * n0, T1 = nm * n1;
  if (P < 2 || T0 + 3 * T1 >= (1 << 20)) return false;
  // ffn2 K splits: 1 by default. (Measured, config (b): 2 splits 104 us and 3
  // splits 163 us vs 75 us unsplit — the ordered partial-sum epilogues chain
  // across pairs.) RTPB_FUSED_SPLITS forces a count (A/B).
  int S = 1;
  if (const char* e = std::getenv("RTPB_FUSED_SPLITS")) S = std::max(1, std::atoi(e));
  TwoProb q;
  q.T0 = T0;
  q.n0 = n0;
  q.c0 = tile_cost(h, 2.0);
  q.T1 = T1;
  q.n1 = n1;
  q.S1 = S;
  q.c1 = S == 1 ? tile_cost(f, 1.0) : tile_cost((f + S - 1) / S, 2.0);
  q.dep = 1;
  plan.est_us = best_schedule(P, q, plan.sched);
  plan.k_splits2 = S;
  if (S == 1 && std::getenv("RTPB_TAIL_SPLIT")) {
    // the final wave's ffn2 tiles split over K in two (ordered partials).
    // Opt-in: measured slower (config (b) forward 96 vs 79 us) — the split
    // units' partial / final epilogues cost more than the tail they trim.
    const double c_half = tile_cost((f + 1) / 2, 2.0);
    for (int tail : {P / 4, P / 2, (3 * P) / 4, P}) {
      if (tail <= 0 || tail > T1) continue;
      for (double al : kAlphas) {
        std::vector<int> s_;
        const double t = list_schedule(P, q, al, s_, nullptr, tail, c_half);
        if (t < plan.est_us) {
          plan.est_us = t;
          plan.sched.swap(s_);
          plan.k_splits2 = 2;
        }
      }
    }
  }
  plan.slots = P;
  plan.dep_rows = nm;
  plan.dep_target = unsigned(n0) * 2u * kEpiWarps;
  plan.tiles2 = T1;
  if (std::getenv("RTPB_DEBUG_PLAN"))
    std::fprintf(stderr, "fused fwd plan: M=%zu h=%zu f=%zu slots=%d splits2=%d est %.1f us\n", M, h, f, P,
                 plan.k_splits2, plan.est_us);
  return true;
}

int gemm_fwd_fused(const StepFwd& p0, const StepFwd& p1, const FusedFwdPlan& plan, const FusedFwdWs& ws,
                   cudaStream_t s) {
  // problem 0: pre = X . W1 + b1 (store_pre) and act = gelu(pre); problem 1: Y = act . W2 + b2
  Op a0{p0.x, nullptr, p0.I, p0.M, p0.ldx}, b0{p0.w, nullptr, p0.per, p0.I, p0.per};
  Op a1{p1.x, nullptr, p1.I, p1.M, p1.ldx}, b1{p1.w, nullptr, p1.per, p1.I, p1.per};
  Out y0{p0.y, false, p0.per, p0.M, p0.ldy}, act0{p0.act, false, p0.per, p0.M, p0.ld_act};
  Out y1{p1.y, false, p1.per, p1.M, p1.ldy};
  const bool split = plan.k_splits2 > 1;
  Out acc1{split ? static_cast<const void*>(ws.acc2) : p1.y, split, p1.per, p1.M, split ? p1.per : p1.ldy};
  GemmMaps m1;
  int rc;
  if ((rc = encode_maps<FusedFwdCfg>(a1, b1, y1, &acc1, m1))) return rc;
  GemmArgs g{};
  g.M = int(p0.M);
  g.N = int(p0.per);
  g.K = int(p0.I);
  g.flags = p0.flags;
  g.aux = p0.bias;
  g.n_fastest = 1;
  g.k_splits = 1;
  g.sched = ws.sched;
  g.M2 = int(p1.M);
  g.N2 = int(p1.per);
  g.K2 = int(p1.I);
  g.flags2 = p1.flags;
  g.aux2 = p1.bias;
  g.n_fastest2 = 1;
  g.k_splits2 = plan.k_splits2;
  g.split_flags2 = ws.split_flags2;
  g.acc2 = ws.acc2;
  g.ld_acc2 = int64_t(p1.per);
  g.dep_count = ws.dep_count;
  g.dep_target = plan.dep_target;
  g.dep_rows = plan.dep_rows;
  g.done_ctas = ws.done_ctas;
  return launch_cfg<FusedFwdCfg>(a0, b0, y0, &act0, g, s, &m1, plan.slots);
}

// ------------------------------------------------------------------ fused MLP backward (N = 1)
// Two concurrent scheduled launches, each on its own CTA-pair slots:
//   D (compute stream, dX config): ffn2's dX with gelu' (dpre, problem 0) then
//     ffn1's dX (problem 1, row block mb after D published dpre row block mb);
//   W (aux stream, dW config): ffn2's dW (problem 0) then ffn1's dW (problem 1,
//     whose K runs over dpre rows: its producer waits per K block on D's
//     row-block counters).
// D never waits on W, and both grids together fit the SMs, so the cross-launch
// waits cannot deadlock; a wait that never completes traps instead of hanging.
namespace {
using FusedDCfg = GemmCfg<EPI_DGRAD, 256, false, kEpiWarps, false, false, true, true>;
using FusedWCfg = GemmCfg<EPI_WGRAD, 256, false, kEpiWarps, true, true, false, true>;

}  // namespace

bool plan_fused_bwd(size_t M, size_t h, size_t f, FusedBwdPlan& plan) {
  const int P = sm_count() / 2;
  const int nm = int((M + 255) / 256);
  const int nd2 = int((f + 255) / 256), nd1 = int((h + 255) / 256);  // dX tiles per row block
  const int Tw = int((f + 255) / 256) * int((h + 255) / 256);       // dW tiles: f x h (ffn2), h x f (ffn1)
  if (P < 4 || nm * (nd2 + nd1) >= (1 << 20)) return false;
  TwoProb d;
  d.T0 = nm * nd2;
  d.n0 = nd2;
  d.c0 = tile_cost(h, 2.0) + 0.6;  // gelu' epilogue streams pre in
  d.T1 = nm * nd1;
  d.n1 = nd1;
  d.c1 = tile_cost(f, 1.0);
  d.dep = 1;
  double best = 1e300;
  // dW K splits: 1. (Measured, config (b): W 127 us unsplit, 146 us with 2
  // ordered splits, 162 us with 3.) RTPB_FUSED_WSPLITS forces a count (A/B).
  int s_lo = 1, s_hi = 1;
  if (const char* e = std::getenv("RTPB_FUSED_WSPLITS")) s_lo = s_hi = std::max(1, std::atoi(e));
  for (int Pw = 2; Pw <= P - 2; ++Pw) {
    const int Pd = P - Pw;
    // D's schedule decides when dpre rows land for W: try every D policy
    // (forward, alpha sweep; the reversed schedule lands rows late) against W
    for (double al : kAlphas) {
    std::vector<int> sd;
    std::vector<double> rows;
    const double td = list_schedule(Pd, d, al, sd, &rows);
    if (td >= best) continue;
    for (int S = s_lo; S <= s_hi; ++S) {
      TwoProb w;
      w.T0 = Tw * S;  // problem 0 (ffn2 dW) units, split-major within a tile via S1 below
      w.n0 = 0;
      w.c0 = tile_cost((M + S - 1) / S, 2.0);
      w.T1 = Tw;
      w.n1 = 0;
      w.S1 = S;
      w.c1 = w.c0;
      w.dep = 2;
      w.ext_ready = &rows;
      w.K1 = M;
      // problem 0 of W is split too: emit its units with split indices
      std::vector<int> sw;
      const double tw = best_schedule(Pw, w, sw);
      const double t = std::max(td, tw);
      if (t < best) {
        best = t;
        // problem-0 codes in sw are plain unit indices u = tile * S + split: re-encode
        for (size_t i = size_t(Pw) + 1; i < sw.size(); ++i)
          if (!(sw[i] >> 28)) sw[i] = ((sw[i] % S) << 20) | (sw[i] / S);
        plan.sched_d = sd;
        plan.sched_w.swap(sw);
        plan.slots_d = Pd;
        plan.slots_w = Pw;
        plan.w_splits = S;
      }
    }
    }
  }
  plan.dep_rows = nm;
  plan.dep_target = unsigned(nd2) * 2u * kEpiWarps;
  plan.est_us = best;
  if (std::getenv("RTPB_DEBUG_PLAN"))
    std::fprintf(stderr, "fused bwd plan: M=%zu h=%zu f=%zu dX pairs %d dW pairs %d (K splits %d) est %.1f us\n", M, h,
                 f, plan.slots_d, plan.slots_w, plan.w_splits, best);
  return true;
}

int gemm_bwd_fused(const FusedBwdArgs& a, const FusedBwdPlan& plan, const FusedBwdWs& ws, cudaStream_t compute,
                   cudaStream_t aux) {
  const size_t M = a.M, h = a.h, f = a.f;
  const unsigned done_target = 2u * unsigned(plan.slots_d + plan.slots_w);
  // ---- D: dpre = (dY . W2^T) * gelu'(pre) over pre; dX = dpre . W1^T
  {
    Op a0{a.dy, nullptr, h, M, a.ldy}, b0{a.w2, nullptr, h, f, h};
    Out dpre{a.pre, false, f, M, f}, pre_in{a.pre, false, f, M, f};
    Op a1{a.pre, nullptr, f, M, f}, b1{a.w1, nullptr, f, h, f};
    Out dx{a.dx, false, h, M, a.lddx};
    GemmMaps m1;
    int rc;
    if ((rc = encode_maps<FusedDCfg>(a1, b1, dx, nullptr, m1))) return rc;
    GemmArgs g{};
    g.M = int(M); g.N = int(f); g.K = int(h);
    g.flags = EF_FIRST | EF_LAST | EF_GELU_BWD | (a.exact_gelu ? EF_EXACT_GELU : 0);
    g.aux = a.pre; g.ld_aux = int64_t(f);
    g.n_fastest = 1; g.k_splits = 1;
    g.sched = ws.sched_d;
    g.M2 = int(M); g.N2 = int(h); g.K2 = int(f);
    g.flags2 = EF_FIRST | EF_LAST;
    g.n_fastest2 = 1; g.k_splits2 = 1;
    g.dep_count = ws.dep_count; g.dep_target = plan.dep_target; g.dep_rows = plan.dep_rows;
    g.done_ctas = ws.done_ctas; g.done_target = done_target;
    if ((rc = launch_cfg<FusedDCfg>(a0, b0, dpre, &pre_in, g, compute, &m1, plan.slots_d))) return rc;
  }
  // ---- W: G2 (+)= act^T . dY ; G1 (+)= X^T . dpre (K blocks after D published them)
  {
    Op a0{a.act, nullptr, f, M, f}, b0{a.dy, nullptr, h, M, a.ldy};
    Out g2{a.g2, true, h, f, h};
    Op a1{a.x, nullptr, h, M, a.ldx}, b1{a.pre, nullptr, f, M, f};
    Out g1{a.g1, true, f, h, f};
    const bool par = plan.w_splits > 1 && a.wpart1 && a.wpart2;
    const size_t fpad = (f + 255) / 256 * 256, hpad = (h + 255) / 256 * 256;
    Out part2{par ? static_cast<const void*>(a.wpart2) : a.g2, true, h, par ? plan.w_splits * fpad : f, h};
    Out part1{par ? static_cast<const void*>(a.wpart1) : a.g1, true, f, par ? plan.w_splits * hpad : h, f};
    GemmMaps m1;
    int rc;
    if ((rc = encode_maps<FusedWCfg>(a1, b1, g1, &part1, m1))) return rc;
    GemmArgs g{};
    g.M = int(f); g.N = int(h); g.K = int(M);
    g.flags = a.g2_zero ? EF_FIRST : 0;
    g.n_fastest = 0; g.k_splits = plan.w_splits; g.split_flags = a.split_flags2;
    g.gbias_in = a.g2_zero ? nullptr : a.g2 + f * h; g.gbias_out = a.g2 + f * h;
    g.bias_part = a.bias_part2; g.bias_tick = a.bias_tick2;
    g.sched = ws.sched_w;
    g.M2 = int(h); g.N2 = int(f); g.K2 = int(M);
    g.flags2 = a.g1_zero ? EF_FIRST : 0;
    g.n_fastest2 = 0; g.k_splits2 = plan.w_splits; g.split_flags2 = a.split_flags1;
    g.gbias_in2 = a.g1_zero ? nullptr : a.g1 + h * f; g.gbias_out2 = a.g1 + h * f;
    g.bias_part2 = a.bias_part1; g.bias_tick2 = a.bias_tick1;
    g.dep_count = ws.dep_count; g.dep_target = plan.dep_target; g.dep_rows = plan.dep_rows; g.dep_on_k = 1;
    g.done_ctas = ws.done_ctas; g.done_target = done_target;
    if (par) {
      g.wpar = 1;
      g.wpart = a.wpart2; g.wpart_rows = int(fpad);
      g.wpart2 = a.wpart1; g.wpart_rows2 = int(hpad);
    }
    if ((rc = launch_cfg<FusedWCfg>(a0, b0, g2, &part2, g, aux, &m1, plan.slots_w))) return rc;
  }
  return RTPB_OK;
}

const void* kernel_anchor_elementwise();
const void* kernel_anchor_attention();
const void* kernel_anchor_moe_embed();

namespace {
template <class T>
T driver_fn(const char* name, int version) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &f, version, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<T>(f);
}
}  // namespace

void preload_device_kernels() {
  static std::mutex mu;
  static unsigned long long done_mask = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard lk(mu);
  if (done_mask >> dev & 1ull) return;
  done_mask |= 1ull << dev;
  static const auto get_module = driver_fn<PFN_cuFuncGetModule_v11000>("cuFuncGetModule", 11000);
  static const auto count_fns = driver_fn<PFN_cuModuleGetFunctionCount_v12040>("cuModuleGetFunctionCount", 12040);
  static const auto enum_fns = driver_fn<PFN_cuModuleEnumerateFunctions_v12040>("cuModuleEnumerateFunctions", 12040);
  static const auto load_fn = driver_fn<PFN_cuFuncLoad_v12040>("cuFuncLoad", 12040);
  // one kernel per translation unit (= module of the fat binary)
  const void* anchors[] = {
      reinterpret_cast<const void*>(&rtp_gemm_kernel<GemmCfg<EPI_FWD, 256, false, kEpiWarps, false, true, false, true>>),
      kernel_anchor_elementwise(), kernel_anchor_attention(), kernel_anchor_moe_embed()};
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    if (cudaGetFuncBySymbol(&f, a) != cudaSuccess || !f) continue;  // (loads that kernel)
    CUmodule mod = nullptr;
    unsigned cnt = 0;
    if (!get_module || !count_fns || !enum_fns || !load_fn || get_module(&mod, reinterpret_cast<CUfunction>(f)) ||
        count_fns(&cnt, mod) || cnt == 0)
      continue;
    std::vector<CUfunction> fns(cnt);
    if (enum_fns(fns.data(), cnt, mod)) continue;
    for (CUfunction fn : fns) load_fn(fn);
  }
  // every step-GEMM instantiation's shared-memory opt-in (launch_cfg)
  set_smem_attr<GemmCfg<0, 128, false, 8, false, true, false, false>>();
  set_smem_attr<GemmCfg<0, 128, false, 8, false, true, false, true>>();
  set_smem_attr<GemmCfg<0, 128, true, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<0, 256, false, 8, false, true, false, false>>();
  set_smem_attr<GemmCfg<0, 256, false, 8, false, true, false, true>>();
  set_smem_attr<GemmCfg<0, 64, false, 8, false, true, false, false>>();
  set_smem_attr<GemmCfg<0, 64, true, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<1, 128, false, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<1, 128, false, 8, false, false, false, true>>();
  set_smem_attr<GemmCfg<1, 128, false, 8, false, false, true, false>>();
  set_smem_attr<GemmCfg<1, 128, true, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<1, 128, true, 8, false, false, true, false>>();
  set_smem_attr<GemmCfg<1, 256, false, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<1, 256, false, 8, false, false, false, true>>();
  set_smem_attr<GemmCfg<1, 256, false, 8, false, false, true, true>>();
  set_smem_attr<GemmCfg<1, 64, false, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<1, 64, true, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<2, 128, false, 8, true, true, false, false>>();
  set_smem_attr<GemmCfg<2, 128, false, 8, true, true, false, true>>();
  set_smem_attr<GemmCfg<2, 128, true, 8, false, false, false, false>>();
  set_smem_attr<GemmCfg<2, 256, false, 8, true, true, false, false>>();
  set_smem_attr<GemmCfg<2, 256, false, 8, true, true, false, true>>();
  set_smem_attr<GemmCfg<2, 64, false, 8, true, true, false, false>>();
  set_smem_attr<GemmCfg<2, 64, true, 8, false, false, false, false>>();
  cudaGetLastError();  // a failed probe leaves no sticky state behind
}

void set_sm_budget(int sms) { t_sm_budget = sms; }
void set_pdl_enabled(bool on) { t_pdl = on; }
void set_launch_wait_flag(const unsigned* flag) { t_wait_flag = flag; }
void set_launch_g_flag(const unsigned* flag) { t_g_flag = flag; }
void set_launch_flag_reset(unsigned* flags, int count, unsigned* ctr) {
  t_reset_flags = flags;
  t_reset_count = flags ? count : 0;
  t_reset_ctr = flags ? ctr : nullptr;
}
int sm_budget() { return sm_count(); }

void set_trace(void* buf, size_t bytes) {
  g_trace = static_cast<unsigned long long*>(buf);
  g_trace_cap = buf ? bytes / sizeof(unsigned long long) : 0;
  g_trace_next = 0;
}

int gemm_fwd(bool f32, const StepFwd& p, cudaStream_t s) {
  // C[M x per] = X[M x I] . W_j[I x per]; A K-major, B MN-major.
  Op a{p.x, p.x_lo, p.I, p.M, p.ldx};
  // bf16: W_j read MN-major in place. tf32: the pre-pass wrote W_j^T (per x I).
  Op b = f32 ? Op{p.w, p.w_lo, p.I, p.per, p.I} : Op{p.w, p.w_lo, p.per, p.I, p.per};
  const size_t esz = f32 ? 4 : 2;
  GemmArgs g{};
  g.M = int(p.M);
  g.N = int(p.per);
  g.K = int(p.I);
  g.flags = p.flags;
  g.aux = p.bias;
  // Output blocks start at column col0 of Y / act: the maps' base pointers.
  Out y{p.y ? static_cast<const char*>(p.y) + p.col0 * esz : nullptr, f32, p.per, p.M, p.ldy};
  Out act{p.act ? static_cast<const char*>(p.act) + p.col0 * esz : nullptr, f32, p.per, p.M, p.ld_act};
  const bool has_y = (p.flags & EF_STORE_PRE) && p.y;
  const bool has_act = (p.flags & EF_GELU) && p.act;
  const Out& c0 = has_y ? y : act;
  return dispatch<EPI_FWD>(f32, a, b, c0, has_act ? &act : nullptr, g, s, p.force_bn);
}

int gemm_dgrad(bool f32, const StepDgrad& p, cudaStream_t s) {
  // C[M x I] = dY_blk[M x per] . W_j^T; A K-major (ld = ldy), B = W_j rows (K-major).
  Op a{p.dy, p.dy_lo, p.per, p.M, p.ldy};
  Op b{p.w, p.w_lo, p.per, p.I, p.per};
  GemmArgs g{};
  g.M = int(p.M);
  g.N = int(p.I);
  g.K = int(p.per);
  struct SegGuard {
    ~SegGuard() { t_kseg = KSeg{}; }
  } seg_guard;
  if (p.w2) {
    // + dY_blk2 . W_2^T: the K loop runs over shard 1 (K blocks padded to 64)
    // then shard 2, one accumulator — two steps' products in one pass.
    if (f32) return set_error(RTPB_ERR_CONFIG, "dgrad over two shards: bf16 only");
    const int kb1 = int((p.per + 63) / 64);
    t_kseg = KSeg{true, kb1, p.dy2, p.w2, p.per, p.M, p.ldy, p.per, p.I, p.per};
    g.K = kb1 * 64 + int(p.per);
  }
  g.flags = p.flags;
  g.aux = p.pre;
  g.ld_aux = int64_t(p.ldpre);
  g.acc = p.acc;
  g.ld_acc = int64_t(p.ld_acc);
  const bool last = p.flags & EF_LAST;
  // last step: emit dX in the activation dtype; otherwise store / reduce-add fp32.
  Out c0 = last ? Out{p.dx, f32, p.I, p.M, p.ldx} : Out{p.acc, true, p.I, p.M, p.ld_acc};
  if (last && (p.flags & EF_GELU_BWD)) {
    // gelu' fused: stream pre tiles through smem (PRE_TMA configs): CTA-pair
    // 256 x 256 tiles (4 stages) when they fill the machine, else 128 x 128.
    Out pre{p.pre, f32, p.I, p.M, p.ldpre};
    int code = p.force_bn ? p.force_bn : choose_tile(g.M, g.N, f32);
    const int bn = (!f32 && code == 1256) ? 256 : 128;
    g.n_fastest = raster_mode(g.M, g.N, g.K, bn == 256 ? 256 : 128, bn, f32, false);
    if (f32) return launch_cfg<GemmCfg<EPI_DGRAD, 128, true, kEpiWarps, false, false, true>>(a, b, c0, &pre, g, s);
    if (bn == 256)
      return launch_cfg<GemmCfg<EPI_DGRAD, 256, false, kEpiWarps, false, false, true, true>>(a, b, c0, &pre, g, s);
    return launch_cfg<GemmCfg<EPI_DGRAD, 128, false, kEpiWarps, false, false, true>>(a, b, c0, &pre, g, s);
  }
  return dispatch<EPI_DGRAD>(f32, a, b, c0, nullptr, g, s, p.force_bn);
}

int gemm_wgrad(bool f32, const StepWgrad& p, cudaStream_t s) {
  // C[I x per] = X^T . dY_blk; bf16: X and dY_blk read MN-major in place.
  // tf32: the pre-pass wrote X^T (I x M) and dY_blk^T (per x M), both K-major.
  const bool kmaj = f32;
  Op a = kmaj ? Op{p.x, p.x_lo, p.M, p.I, p.ldx} : Op{p.x, p.x_lo, p.I, p.M, p.ldx};
  Op b = kmaj ? Op{p.dy, p.dy_lo, p.M, p.per, p.ldy} : Op{p.dy, p.dy_lo, p.per, p.M, p.ldy};
  GemmArgs g{};
  g.M = int(p.I);
  g.N = int(p.per);
  g.K = int(p.M);
  // G_out = G_in + P: the epilogue reduce-adds into G_out, so seed it with G_in.
  // G_in == nullptr: G is known zero, the first split stores instead.
  g.flags = p.g_in ? 0 : EF_FIRST;
  if (p.g_in && p.g_out != p.g_in) {
    cudaError_t e = cudaMemcpyAsync(p.g_out, p.g_in, p.I * p.per * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return set_cuda_error(e, "wgrad: seed G_out");
  }
  Out c0{p.g_out, true, p.per, p.I, p.per};
  g.split_flags = p.split_flags;
  g.gbias_in = p.gbias_in;
  g.gbias_out = p.gbias_out;
  g.bias_part = p.bias_part;
  g.bias_tick = p.bias_tick;
  int par = 0;
  if (p.wpart && !f32) {
    // unordered partials + slice folds for long split chains (see
    // wgrad_partial_floats); RTPB_WGRAD_PAR forces a mode (0 = the chain)
    GemmArgs t = g;
    pick_code<EPI_WGRAD>(false, t, p.force_bn);
    const char* e = std::getenv("RTPB_WGRAD_PAR");
    par = e ? std::atoi(e) : (t.k_splits >= kParMinSplits ? 2 : 0);
    if (t.k_splits < 2) par = 0;
  }
  if (par) {
    // split-K partials: one (I rounded up to 256) x per fp32 block per split
    const size_t ipad = (p.I + 255) / 256 * 256;
    const int smax = wgrad_splits(f32, p.M, p.I, p.per, p.force_bn);
    Out part{p.wpart, true, p.per, size_t(smax) * ipad, p.per};
    // every unit of a split dW launch is resident (splits <= pairs / tiles):
    // 2 = parallel slice folds, 1 = the last arriver folds
    g.wpar = par == 1 ? 1 : 2;
    g.wpart = p.wpart;
    g.wpart_rows = int(ipad);
    g.gout = p.g_out;
    return dispatch<EPI_WGRAD>(f32, a, b, c0, &part, g, s, p.force_bn);
  }
  return dispatch<EPI_WGRAD>(f32, a, b, c0, nullptr, g, s, p.force_bn);
}

int wgrad_splits(bool f32, size_t M, size_t I, size_t per, int force_bn) {
  GemmArgs g{};
  g.M = int(I);
  g.N = int(per);
  g.K = int(M);
  unsigned dummy = 0;
  g.split_flags = &dummy;
  // the most splits any SM budget can ask for (workspace sizing): the
  // split-to-fill choice grows with the budget, the wave-quantisation one
  // does not, so every budget is evaluated
  const int saved = t_sm_budget;
  int most = 1;
  for (int b = device_sms(); b >= 2; b -= 2) {
    t_sm_budget = b;
    GemmArgs t = g;
    pick_code<EPI_WGRAD>(f32, t, force_bn);
    most = std::max(most, t.k_splits);
  }
  t_sm_budget = saved;
  return most;
}

size_t wgrad_partial_floats(bool f32, size_t M, size_t I, size_t per) {
  // Split-K partials for the unordered dW mode (every split stores its fp32
  // partial, then folds a row slice of all of them into G in split order:
  // deterministic). The ordered chain pays one epilogue + hand-off per split
  // in sequence, the partials a store and a fold: the chain wins for short
  // chains (config (b) N = 4, 3-4 splits: 440 vs 379 TFLOP/s per GPU), the
  // partials for long ones (N = 8, 5-8 splits: 250 vs 243), so they are used
  // from kParMinSplits splits. RTPB_WGRAD_PAR forces a mode (0 = the chain,
  // 1 = the last arriver folds, 2 = slice folds).
  if (f32) return 0;
  const char* mode = std::getenv("RTPB_WGRAD_PAR");
  if (mode && std::atoi(mode) == 0) return 0;
  const int S = wgrad_splits(f32, M, I, per, 0);
  if (!mode && S < kParMinSplits) return 0;
  return S > 1 ? size_t(S) * ((I + 255) / 256 * 256) * per : 0;
}

bool wgrad_fuses_bias(bool f32, size_t M, size_t I, size_t per, unsigned* split_flags, int force_bn) {
  GemmArgs g{};
  g.M = int(I);
  g.N = int(per);
  g.K = int(M);
  g.split_flags = split_flags;
#ifdef RTPB_NO_COLSUM
  return false;
#endif
  return !f32 && pick_code<EPI_WGRAD>(false, g, force_bn) > 1000;
}

}  // namespace rtpb
