// Persistent, warp-specialised tcgen05 GEMM for the three per-rotation-step
// products of an RTP linear (layers_linear.cpp:35, :61, :65):
//
//   FWD   : Y[:, col0 + n] = X . W_j + b_j        A = X (K-major), B = W_j (MN-major)
//           (+ optional exact-erf GELU: writes pre and gelu(pre))
//   DGRAD : dXacc += dY[:, blk_j] . W_j^T         A = dY blk (K-major), B = W_j (K-major)
//           (fp32 cross-step accumulator; last step casts, optionally * gelu'(pre))
//   WGRAD : G += X^T . dY[:, blk_j]               A = X (MN-major), B = dY blk (MN-major)
//           (the travelling gradient shard is accumulated by the epilogue)
//
// Roles (one CTA per SM, grid = min(tiles, SMs), static round-robin tiles):
//   warp 0        : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1        : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..2+E  : epilogue: TMEM -> registers -> swizzled smem staging ->
//                   TMA store (bf16 / fp32) or TMA reduce-add (fp32, done in
//                   L2: the dX cross-step accumulation and G += dW never make
//                   the SMs read the accumulator). Double-buffered TMEM
//                   accumulators overlap tile t's epilogue with tile t+1's MMAs.
// Tile: BM = 128 rows (UMMA M=128, cta_group::1) x BN columns, BK = 128 bytes
// of K per stage (64 bf16 / 32 fp32), SWIZZLE_128B operands.
// TF32X3: fp32 operands split (and, where the GEMM would read them MN-major,
// transposed to K-major) by a pre-pass into hi (low 13 mantissa bits zeroed)
// and lo = x - hi; D += Ahi.Bhi + Ahi.Blo + Alo.Bhi on kind::tf32.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

namespace rtpb {

enum EpiKind : int { EPI_FWD = 0, EPI_DGRAD = 1, EPI_WGRAD = 2 };
enum EpiFlags : int {
  EF_GELU = 1,      // FWD: also emit gelu(pre) through map c1
  EF_FIRST = 2,     // DGRAD: first step (accumulator not read)
  EF_LAST = 4,      // DGRAD: last step (emit the cast result through map c0)
  EF_GELU_BWD = 8,  // DGRAD last step: multiply by gelu'(pre)
  EF_STORE_PRE = 16, // FWD: store pre through map c0
  EF_EXACT_GELU = 64 // bf16: exact-erf GELU / GELU' instead of the tanh.approx form
};

struct GemmArgs {
  int M, N, K;
  int flags;
  int n_fastest;       // tile raster: 0 m fastest, 1 n fastest (A streamed once), >= 2 grouped (that many row blocks)
  const void* aux;     // FWD: bias (dtype, N values) | DGRAD: pre (dtype, M x N, ld_aux)
  int64_t ld_aux;
  const float* acc;    // DGRAD LAST && !FIRST: fp32 accumulator read (M x N, ld_acc)
  int64_t ld_acc;
  // WGRAD split-K: work unit = (tile, split); split s reduce-adds its partial
  // into G only after split s-1 of the same tile has completed its writes
  // (per-tile counter in zeroed workspace, reset by the last split), so the
  // summation order is fixed and results are bitwise reproducible.
  int k_splits;
  unsigned* split_flags;
  // WGRAD CTA-pair path: the bias gradient db = colsum(dY block) is fused —
  // an extra warp sums the dY tiles staged in smem as the B operand.
  const float* gbias_in;  // nullable: gradient known zero
  float* gbias_out;
  float* bias_part;       // [ceil(M / 256) * k_splits][N] partial sums
  unsigned* bias_tick;    // [ceil(N / 64)] zeroed, self-resetting arrival counters
  // Debug timeline (nullable; rtpb_debug_trace): per CTA TRACE_STRIDE u64 of
  // %globaltimer stamps: [0] entry, [1] after griddep_wait, then per local
  // work unit i < TRACE_UNITS at 2 + 6 i: MMA starts waiting for a free
  // accumulator, accumulator free, first stage landed, last MMA committed,
  // epilogue sees the accumulator, epilogue released it; last slot = gridDim.x.
  unsigned long long* trace;
  // Scheduled multi-problem launch (nullable sched: static round-robin over
  // problem 0's units). Unit slot s (a CTA pair, or a CTA) processes the units
  // sched[sched[s] .. sched[s + 1]), each encoded prob << 28 | split << 20 |
  // tile, in that order. Problem 1 (same kernel config, its maps in the second
  // GemmMaps) has geometry M2 x N2 x K2 and epilogue flags2 / aux2; its tile
  // row block mb may start loading only when dep_count[mb] >= dep_target,
  // which problem 0's epilogue warps advance (one arrival per warp per tile
  // of that row block) once their stores of the tile are complete. The last
  // CTA to finish re-zeroes dep_count[0 .. dep_rows) and done_ctas.
  const int* sched;
  int M2, N2, K2, flags2, n_fastest2;
  const void* aux2;
  // Problem 1 split over K (FWD only): split s < k_splits2 - 1 stores (s = 0)
  // or reduce-adds its fp32 partial into acc2 (M2 x N2, map c1 of the second
  // GemmMaps), in split order via split_flags2[tile]; the last split adds
  // acc2, the bias and writes the output. Deterministic.
  int k_splits2;
  unsigned* split_flags2;
  const float* acc2;
  int64_t ld_acc2;
  // Problem 1 of a dW launch: its own fused bias-gradient sums.
  const float* gbias_in2;
  float* gbias_out2;
  float* bias_part2;
  unsigned* bias_tick2;
  // dep_on_k: problem 1's K dimension runs over the rows another (concurrent)
  // launch publishes: its producer waits per K block on
  // dep_count[k_row / 256] instead of per tile row block. done_target: CTAs
  // sharing dep_count / done_ctas across launches (0: this grid).
  int dep_on_k;
  unsigned done_target;
  // dW split over K without an ordered chain (wpar): every split stores its
  // fp32 partial into map c1 (rows split * wpart_rows + row, wpart_rows = M
  // rounded up to the tile height) and counts in on its region's counter
  // (split_flags[tile * 16 + warp slot]); the warp that completes a region sums
  // the partials in split order and adds them into G once. Deterministic.
  int wpar;  // 1: the last split folds; 2: all splits resident, each folds a row slice
  int wpart_rows, wpart_rows2;
  const float* wpart;
  const float* wpart2;
  float* gout;  // wpar 2: the gradient block written by plain stores (I x per, ld per)
  float* gout2;
  // Operand arrival written by another stream (the rotation's comm stream,
  // cuStreamWriteValue32): the producers load nothing before *ready_flag >= 1.
  // Replaces a stream-event dependency, so the launch keeps its programmatic
  // (PDL) edge to the previous GEMM on its stream.
  const unsigned* ready_flag;
  // WGRAD: the travelling gradient shard G arrives by flag (comm stream,
  // cuStreamWriteValue32 once the neighbour's G has landed). Only the roles
  // that read or reduce into G wait for *g_flag >= 1 — the epilogue warps
  // before their first tile's G update, the bias-sum warps before adding
  // G's bias part — so the producer and MMA run the mainloop while G is in
  // flight: the accumulation is applied in the epilogue as the shard arrives.
  const unsigned* g_flag;
  // Two K segments (DGRAD over two resident weight shards, single problem):
  // K blocks kb >= kseg_kb read the A and B maps of the second GemmMaps at
  // K offset (kb - kseg_kb) * BK. 0: one segment.
  int kseg_kb;
  // The last reader of a pass's arrival flags clears them: once every CTA of
  // this grid is done (counter flag_reset_ctr), [flag_reset, +flag_reset_count)
  // and the counter return to 0. Every flag of the pass was set before this
  // grid passed its own flag wait (one comm stream, in order), and the next
  // pass's readers run after this grid (stream order / griddepcontrol.wait).
  unsigned* flag_reset;
  unsigned* flag_reset_ctr;
  int flag_reset_count;
  unsigned* dep_count;
  unsigned dep_target;
  int dep_rows;
  unsigned* done_ctas;
  // Pass launch (pass_steps = S > 0; FWD or DGRAD, one problem, no split-K):
  // every rotation step of one layer pass in ONE persistent launch, so the
  // N small step GEMMs of a ring pass pay one prologue and no launch gaps, and
  // a tile's epilogue overlaps the next tile's MMAs across step boundaries.
  // Work unit = (step s, tile t); slot k runs its tiles t = k, k + slots, ...
  // for s = 0, 1, ... in order. Step s reads its weight shard through maps.b
  // (bit s of pass_buf clear) or maps2.b (set): the resident shard and the
  // out-of-place spare alternate.
  //   FWD  : output at column pass_col[s] + n of the full-width maps c0 / c1
  //          (the shard's column block j * per); bias from aux (buffer 0) or
  //          aux2 (buffer 1). Requires per % 32 == 0 (32-column store boxes).
  //   DGRAD: A (dY) read from column pass_col[s]; step 0 stores the fp32
  //          accumulator (maps.c0), middle steps reduce-add into it, the last
  //          loads it and writes dX through maps2.c0. A tile's successive
  //          steps run on the same slot and warps, which drain their bulk
  //          reductions at every step boundary: the summation order is the
  //          step order, as with one launch per step.
  // Step s >= 1 loads nothing before pass_ready[s] >= 1 (the comm stream's
  // arrival flag). Once a tile's MMAs completed (its operands were read),
  // every epilogue warp counts in on pass_done[g] (g: the unit's group, see
  // pass_pair): the comm stream waits for tiles x warps there
  // (cuStreamWaitValue32) before it lands a later shard in the group's
  // buffers. The grid's last CTA re-zeroes pass_done.
  // pass_pair (DGRAD): a unit covers the step pair (2g, 2g + 1) as two K
  // segments — buffer 0 at dY column pass_col[2g], then buffer 1 at
  // pass_col[2g + 1] — one accumulation over K = 2 per (paired dX: half the
  // fp32 accumulator passes).
  //   WGRAD: G += X^T dY[:, pass_col[s] :] for every step into the ONE
  //          travelling gradient buffer (units (tile, split) of step s per
  //          slot, ordered split-K chain within a step). pass_ready[s] is G's
  //          arrival flag: only the epilogue waits for it (the mainloops of
  //          step s run while G(s) is in flight), and every epilogue warp
  //          counts in on pass_done[s] once its reductions of the unit have
  //          LANDED — the comm stream then sends G on. The bias part: the
  //          warp of unit (tile 0, split 0) adds pass_db[pass_col[s] + c]
  //          (dY's column sums, computed once for the pass) into
  //          pass_gbias[c] after G(s) landed. EF_FIRST (args.flags): G is known
  //          zero at step 0 (stores instead of reduce-adds).
  int pass_steps;
  int pass_pair;
  unsigned pass_buf;
  int pass_col[16];
  const unsigned* pass_ready;
  unsigned* pass_done;
  const float* pass_db;
  float* pass_gbias;
};
constexpr int TRACE_UNITS = 12;  // 2 + 6 * 12 slots + grid marker at TRACE_STRIDE - 1
constexpr int TRACE_STRIDE = 80;

template <int EPI_, int BN_, bool TF32_, int EPI_WARPS_, bool A_MN_, bool B_MN_, bool PRE_TMA_ = false,
          bool PAIR_ = false>
struct GemmCfg {
  static constexpr int EPI = EPI_;
  // PAIR: a CTA pair (cluster of 2) computes a 256 x BN tile with
  // tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and half
  // of B's BN columns, the leader issues the MMAs, each CTA's TMEM holds its
  // 128 accumulator rows. Halves per-SM smem traffic for B.
  static constexpr bool PAIR = PAIR_;
  static constexpr int TILE_M = PAIR ? 256 : 128;
  static constexpr int B_ROWS = PAIR ? BN_ / 2 : BN_;  // B rows (N) staged per CTA
  // DGRAD with gelu' fused: the tile's pre values are streamed into shared
  // memory by TMA when the tile starts (while its MMAs run), instead of
  // per-row global loads in the epilogue.
  static constexpr bool PRE_TMA = PRE_TMA_;
  static constexpr int BM = 128;
  static constexpr int BN = BN_;
  static constexpr bool TF32 = TF32_;
  static constexpr int ELEM = TF32 ? 4 : 2;
  static constexpr int BK = 128 / ELEM;          // K elements per stage
  static constexpr int UMMA_K = 32 / ELEM;       // 16 bf16 / 8 tf32
  static constexpr int KSTEPS = BK / UMMA_K;     // 4
  static constexpr int ATOM_MN = 128 / ELEM;     // MN elements per 128B swizzle row
  static constexpr bool A_MN = A_MN_;  // bf16: FWD (K,MN), DGRAD (K,K), WGRAD (MN,MN)
  static constexpr bool B_MN = B_MN_;  // tf32: always (K,K) — operands pre-transposed
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = B_ROWS * 128;
  static constexpr int NOPS = TF32 ? 2 : 1;      // hi (+ lo) copies per operand
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int EPI_WARPS = EPI_WARPS_;
  // Epilogue staging per warp: one 32 x 32 tile per output. FWD writes two
  // outputs (pre, gelu(pre)) in the activation dtype; DGRAD may stage fp32
  // (accumulator steps), WGRAD always does.
  static constexpr int NOUT = EPI == EPI_FWD ? 2 : 1;
  static constexpr int STG_ONE = 32 * 32 * (EPI == EPI_FWD ? ELEM : 4);
  // dW: two fp32 staging buffers per warp, so a chunk's reduce-add into the
  // travelling gradient is in flight while the next chunk is staged.
#ifdef RTPB_WGRAD_STG1
  static constexpr int STG_BUFS = NOUT;
#else
  static constexpr int STG_BUFS = EPI == EPI_WGRAD ? 2 : NOUT;
#endif
  static constexpr int STG_WARP = STG_BUFS * STG_ONE;
  static constexpr int STG_BYTES = EPI_WARPS * STG_WARP;
  // PRE_TMA: every chunk (32 x 32 tile, activation dtype) a warp handles in one tile.
  static constexpr int PRE_CHUNKS = BN / 32 / (EPI_WARPS / 4);
  static constexpr int PRE_WARP = PRE_TMA ? PRE_CHUNKS * 32 * 32 * ELEM : 0;
  static constexpr int PRE_BYTES = EPI_WARPS * PRE_WARP;
  // FWD: each warp's bias slice for a tile (fp32), fetched before the
  // accumulator wait so the loads overlap the tile's MMAs.
  static constexpr int BIAS_WARP = EPI == EPI_FWD ? PRE_CHUNKS * 32 * 4 : 0;
  static constexpr int BIAS_BYTES = EPI_WARPS * BIAS_WARP;
  // dW on CTA pairs: two more warps compute the bias gradient db = colsum(dY)
  // from the B (dY) tiles already staged for the MMA — no second read of dY.
  // Each takes half of a stage's K rows; their sums meet in COLSUM_BYTES.
  // (Measured, config (b) dW in the step graph: 45.5 us per launch vs 42.4 us
  // for the GEMM alone; the stand-alone column-sum kernel cost ~6 us more.)
#ifdef RTPB_NO_COLSUM
  static constexpr bool COLSUM = false;
#else
  static constexpr bool COLSUM = EPI == EPI_WGRAD && PAIR && !TF32;
#endif
  static constexpr int COLSUM_WARPS = COLSUM ? 2 : 0;
  static constexpr int COLSUM_BYTES = COLSUM ? B_ROWS * 4 : 0;
  static constexpr int SMEM_LIMIT = 232448;     // 227 KB opt-in per block
  static constexpr int RESERVE =
      1024 /*align*/ + 512 /*barriers*/ + STG_BYTES + PRE_BYTES + BIAS_BYTES + COLSUM_BYTES;
  static constexpr int STAGES_RAW = (SMEM_LIMIT - RESERVE) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int THREADS = 64 + 32 * (EPI_WARPS + COLSUM_WARPS);
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + RESERVE;
  static constexpr uint32_t IDESC = ptx::idesc_make(TILE_M, BN, TF32 ? 2 : 1, A_MN, B_MN);
  static_assert(!PAIR || (!TF32 && (!B_MN || B_ROWS % ATOM_MN == 0)), "pair tiles: bf16, B halves in whole atoms");
  static_assert(STAGES >= 2, "not enough shared memory for 2 stages");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "epilogue warps");
};

// a, b (+ lo parts): operand loads. c0, c1: epilogue stores / reductions,
// box 32 x 32 (SWIZZLE_64B for bf16 rows of 64 B, SWIZZLE_128B for fp32).
//   FWD   c0 = pre / Y (dtype), c1 = gelu(pre) (dtype)
//   DGRAD c0 = dX (dtype) when EF_LAST, else the fp32 accumulator
//   WGRAD c0 = G (fp32, reduce-add)
struct GemmMaps {
  CUtensorMap a, b, a_lo, b_lo, c0, c1;
};
// (DGRAD + PRE_TMA: c1 is the load map of pre, same 32 x 32 boxes as c0.)

namespace detail {

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_at(unsigned long long* tr, int slot) {
  if (tr) tr[blockIdx.x * TRACE_STRIDE + slot] = gtime();
}

// Spin until *p >= need (acquire, gpu scope), then order async-proxy (TMA)
// accesses after it. A wait that cannot be satisfied within ~10 s traps
// (kernel error) instead of hanging the device.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// RTPB_HANG_DEBUG builds report the expired counter first (a printf costs
// every instantiation a stack frame, so release builds only trap).
__device__ __forceinline__ void wait_expired(const unsigned* p, unsigned need) {
#ifdef RTPB_HANG_DEBUG
  printf("rtpb: bounded wait expired: block %d thread %d counter %p holds %u, needs %u\n", int(blockIdx.x),
         int(threadIdx.x), static_cast<const void*>(p), ld_acquire(p), need);
#endif
  __trap();
}
__device__ __forceinline__ void wait_counter_nofence(const unsigned* p, unsigned need) {
  const long long t0 = clock64();
  while (ld_acquire(p) < need)
    if (clock64() - t0 > (20ll << 30)) wait_expired(p, need);
}
__device__ __forceinline__ void wait_counter(const unsigned* p, unsigned need) {
  wait_counter_nofence(p, need);
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
// a += lo(u), b += hi(u) for a packed bf16 pair (exact widening, fp32 add RN).
// (Shift / mask + FADD: the mixed-precision FHADD.BF16 form measured far slower.)
__device__ __forceinline__ void acc_bf16x2(float& a, float& b, uint32_t u) {
  a += __uint_as_float(u << 16);
  b += __uint_as_float(u & 0xFFFF0000u);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Exact-erf GELU (tensor.cpp:323-351) in the epilogue, evaluated as
// Phi(x) = 0.5 * (1 + erf(x / sqrt2)) with the Abramowitz-Stegun 7.1.26 form
// erf(z) = 1 - P(t) exp(-z^2), t = 1 / (1 + p z), |error| <= 1.5e-7, so that
// GELU and its derivative share one exponential exp(-x^2/2) (which is also
// sqrt(2 pi) * phi(x)): two MUFU ops and ~12 FMAs instead of libdevice erff's
// two-branch polynomial. The error is ~100x below bf16 resolution and below
// the fp32 mode's 1e-5 tolerance.
__device__ __forceinline__ void gelu_parts(float x, float& cdf, float& pdf) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = __fdividef(1.0f, fmaf(0.3275911f, z, 1.0f));
  const float e = __expf(-0.5f * x * x);
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float tail = 0.5f * p * e;  // 0.5 * (1 - erf(z))
  cdf = x >= 0.f ? 1.0f - tail : tail;
  pdf = 0.39894228040143267794f * e;
}
// bf16 mode: GELU in its tanh form with the hardware tanh (one MUFU op):
// |gelu_tanh - gelu_erf| <= ~3e-4 over the real line, below the bf16 output
// resolution (and 100x inside the 2e-2 tolerance); ~6 instructions/element
// instead of ~16, which is what the epilogue's issue rate is bound by.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <bool ACCURATE>
__device__ __forceinline__ float gelu_f(float x) {
  if constexpr (ACCURATE) {
    float c, d;
    gelu_parts(x, c, d);
    return x * c;
  } else {
    const float x2 = x * x;
    const float u = x * fmaf(0.0356774081f, x2, 0.7978845608f);  // sqrt(2/pi) (x + 0.044715 x^3)
    const float hx = 0.5f * x;
    return fmaf(hx, tanh_fast(u), hx);
  }
}
template <bool ACCURATE>
__device__ __forceinline__ float gelu_grad_f(float x) {
  if constexpr (ACCURATE) {
    float c, d;
    gelu_parts(x, c, d);
    return fmaf(x, d, c);
  } else {
    const float x2 = x * x;
    const float u = x * fmaf(0.0356774081f, x2, 0.7978845608f);
    const float t = tanh_fast(u);
    const float du = fmaf(0.1070322243f, x2, 0.7978845608f);  // d u / d x
    // 0.5 (1 + t) + 0.5 x (1 - t^2) du
    return fmaf(0.5f * x * du, fmaf(-t, t, 1.0f), fmaf(0.5f, t, 0.5f));
  }
}

// Load 8 consecutive values of the activation dtype as fp32.
template <bool F32>
__device__ __forceinline__ void load8(const void* base, int64_t off, float* o) {
  if constexpr (F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    float4 a = p[0], b = p[1];
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  } else {
    uint4 u = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off);
    o[0] = bf16lo(u.x); o[1] = bf16hi(u.x); o[2] = bf16lo(u.y); o[3] = bf16hi(u.y);
    o[4] = bf16lo(u.z); o[5] = bf16hi(u.z); o[6] = bf16lo(u.w); o[7] = bf16hi(u.w);
  }
}

// Thread `row` (0..31) writes its 32 values into a 32x32 staging tile laid
// out as the TMA box expects: bf16 rows of 64 B under SWIZZLE_64B (16 B
// chunk c -> c ^ ((row >> 1) & 3)), fp32 rows of 128 B under SWIZZLE_128B
// (chunk c -> c ^ (row & 7)). Conflict-free for 16-byte stores.
template <bool F32OUT>
__device__ __forceinline__ void stage_row(uint8_t* stg, int row, const float* v) {
  if constexpr (F32OUT) {
    uint8_t* base = stg + row * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int pc = c ^ (row & 7);
      *reinterpret_cast<float4*>(base + pc * 16) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
  } else {
    uint8_t* base = stg + row * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int pc = c ^ ((row >> 1) & 3);
      uint4 u;
      u.x = pack_bf16(v[8 * c + 0], v[8 * c + 1]);
      u.y = pack_bf16(v[8 * c + 2], v[8 * c + 3]);
      u.z = pack_bf16(v[8 * c + 4], v[8 * c + 5]);
      u.w = pack_bf16(v[8 * c + 6], v[8 * c + 7]);
      *reinterpret_cast<uint4*>(base + pc * 16) = u;
    }
  }
}

// Inverse of stage_row: thread `row` reads its 32 values from a swizzled tile.
template <bool F32IN>
__device__ __forceinline__ void unstage_row(const uint8_t* stg, int row, float* v) {
  if constexpr (F32IN) {
    const uint8_t* base = stg + row * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 f = *reinterpret_cast<const float4*>(base + (c ^ (row & 7)) * 16);
      v[4 * c] = f.x; v[4 * c + 1] = f.y; v[4 * c + 2] = f.z; v[4 * c + 3] = f.w;
    }
  } else {
    const uint8_t* base = stg + row * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 u = *reinterpret_cast<const uint4*>(base + (c ^ ((row >> 1) & 3)) * 16);
      v[8 * c + 0] = bf16lo(u.x); v[8 * c + 1] = bf16hi(u.x);
      v[8 * c + 2] = bf16lo(u.y); v[8 * c + 3] = bf16hi(u.y);
      v[8 * c + 4] = bf16lo(u.z); v[8 * c + 5] = bf16hi(u.z);
      v[8 * c + 6] = bf16lo(u.w); v[8 * c + 7] = bf16hi(u.w);
    }
  }
}

}  // namespace detail

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    rtp_gemm_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ GemmMaps maps2,
                    const __grid_constant__ GemmArgs args) {
  using namespace ptx;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr bool F32 = Cfg::TF32;  // activation / output dtype is fp32 in TF32 mode

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Align by offsetting smem_raw itself (not through an integer cast) so the
  // compiler keeps the shared address space: STS/LDS instead of generic ST/LD.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage_base = smem;
  uint8_t* stg_base = smem + STAGES * Cfg::STAGE_BYTES;  // 1024-aligned (stage bytes are multiples of 1 KB)
  uint8_t* pre_base = stg_base + Cfg::STG_BYTES;
  float* bias_base = reinterpret_cast<float*>(pre_base + Cfg::PRE_BYTES);
  float* csum_base = bias_base + Cfg::BIAS_BYTES / 4;  // COLSUM: [B_ROWS] partial sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(pre_base + Cfg::PRE_BYTES + Cfg::BIAS_BYTES + Cfg::COLSUM_BYTES);
  uint64_t* full_bar = bars;                    // [STAGES]
  uint64_t* empty_bar = bars + STAGES;          // [STAGES]
  uint64_t* tfull_bar = bars + 2 * STAGES;      // [2]
  uint64_t* tempty_bar = bars + 2 * STAGES + 2; // [2]
  uint64_t* pre_bar = bars + 2 * STAGES + 4;    // [EPI_WARPS] (PRE_TMA)
  uint64_t* ready_bar = pre_bar + Cfg::EPI_WARPS;  // [STAGES] (COLSUM): stage landed, both CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready_bar + (Cfg::COLSUM ? STAGES : 0));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // Pair mode: both CTAs of a cluster work on the same 256-row tile.
  const uint32_t rank = Cfg::PAIR ? cluster_ctarank() : 0;
  const int unit = Cfg::PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int units = Cfg::PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
  const int num_m = (args.M + Cfg::TILE_M - 1) / Cfg::TILE_M;
  const int num_n = (args.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (args.K + BK - 1) / BK;
  // Work unit u = split * num_tiles + tile: every split-s unit precedes every
  // split-(s+1) unit in each CTA's sequence, so the ordered reduction below
  // always waits on work that is running or done (no deadlock).
  const int splits = args.k_splits > 1 ? args.k_splits : 1;
  const int num_units = num_tiles * splits;
  const int kb_per = (num_kb + splits - 1) / splits;
  // This slot's unit sequence: a static round-robin over problem 0, or its
  // list in the scheduled multi-problem launch.
  int it_beg = unit, it_end = num_units, it_step = units;
  if (args.sched) {
    it_beg = __ldg(args.sched + unit);
    it_end = __ldg(args.sched + unit + 1);
    it_step = 1;
  }
  // pass launch: iteration it -> (step, tile). DGRAD: this slot's tiles
  // (t = unit + k * units) step by step, so a tile's steps run on one slot in
  // order. FWD (no cross-step state): the flat (step, tile) sequence over all
  // slots, so a pass with fewer tiles per step than slots still fills them.
  const bool pass = args.pass_steps > 0;
  const bool pass_flat = pass && Cfg::EPI == EPI_FWD;
  const int pass_nt = pass ? (num_units - unit + units - 1) / units : 0;  // per-step units (tile, split)
  const int pass_groups = args.pass_pair ? (args.pass_steps + 1) / 2 : args.pass_steps;
  if (pass_flat) {
    it_beg = unit;
    it_end = pass_groups * num_tiles;
    it_step = units;
  } else if (pass) {
    it_beg = 0;
    it_end = pass_groups * pass_nt;
    it_step = 1;
  }
  const int num_m2 = (args.M2 + Cfg::TILE_M - 1) / Cfg::TILE_M;
  const int num_n2 = (args.N2 + BN - 1) / BN;
  const int num_kb2 = (args.K2 + BK - 1) / BK;
  const int splits2 = args.k_splits2 > 1 ? args.k_splits2 : 1;
  const int kb_per2 = (num_kb2 + splits2 - 1) / splits2;
  struct Unit {
    int prob, t, mb, nb, split, kb0, kb1, M, N, flags;
    bool whole;  // problem 1 of a split launch run unsplit (split code 0xFF)
    int step;    // pass launch: rotation step, or step pair (pass_pair) (else 0)
    bool buf1;   // pass launch: the step's shard is in buffer 1 (maps2.b / aux2)
    int seg_kb;  // pass_pair: K blocks of the first step (the second step's start); 0 = one step
  };
  auto decode = [&](int it) {
    Unit x;
    x.step = 0;
    x.buf1 = false;
    x.seg_kb = 0;
    if (pass) {
      x.prob = 0;
      x.step = pass_flat ? it / num_tiles : it / pass_nt;
      const int u = pass_flat ? it % num_tiles : unit + (it % pass_nt) * units;
      x.split = u / num_tiles;  // split-major within a step (WGRAD split-K)
      x.t = u % num_tiles;
      x.buf1 = !args.pass_pair && ((args.pass_buf >> x.step) & 1u);
    } else if (args.sched) {
      const int e = __ldg(args.sched + it);
      x.prob = e >> 28;
      x.split = (e >> 20) & 0xFF;
      x.t = e & 0xFFFFF;
    } else {
      x.prob = 0;
      x.t = it % num_tiles;
      x.split = it / num_tiles;
    }
    const int nm = x.prob ? num_m2 : num_m, nn = x.prob ? num_n2 : num_n;
    const int nf = x.prob ? args.n_fastest2 : args.n_fastest;
    if (nf >= 2) {
      // grouped raster: nf row blocks at a time, n fastest within the group,
      // so the concurrent tiles share a few A row panels and B column panels
      const int first_m = (x.t / (nf * nn)) * nf;
      const int gsz = min(nm - first_m, nf);
      const int r = x.t % (nf * nn);
      x.mb = first_m + r % gsz;
      x.nb = r / gsz;
    } else if (nf) {
      x.nb = x.t % nn;
      x.mb = x.t / nn;
    } else {
      x.mb = x.t % nm;
      x.nb = x.t / nm;
    }
    x.whole = false;
    if (x.prob && x.split == 0xFF) {
      x.whole = true;
      x.split = 0;
      x.kb0 = 0;
      x.kb1 = num_kb2;
    } else if (x.prob) {
      x.kb0 = x.split * kb_per2;
      x.kb1 = min(num_kb2, x.kb0 + kb_per2);
    } else {
      x.kb0 = x.split * kb_per;
      x.kb1 = min(num_kb, x.kb0 + kb_per);
    }
    x.M = x.prob ? args.M2 : args.M;
    x.N = x.prob ? args.N2 : args.N;
    x.flags = x.prob ? args.flags2 : args.flags;
    if (pass && Cfg::EPI == EPI_WGRAD) {  // G known zero at step 0 only
      if (x.step > 0) x.flags &= ~EF_FIRST;
    } else if (pass) {  // DGRAD: the pass's first step stores the accumulator, its last emits dX
      x.flags &= ~(EF_FIRST | EF_LAST);
      if (x.step == 0) x.flags |= EF_FIRST;
      if (x.step == pass_groups - 1) x.flags |= EF_LAST;
      if (args.pass_pair && 2 * x.step + 1 < args.pass_steps) {
        x.seg_kb = num_kb;
        x.kb1 = 2 * num_kb;
      }
    }
    return x;
  };

  // The bias column-sum warps take part in the stage pipeline only when a
  // launch asks for the bias gradient (a launch without it — a pass launch,
  // a projection, a separately summed bias — runs as if they were absent).
  const bool colsum_live = Cfg::COLSUM && (args.gbias_out != nullptr || args.gbias_out2 != nullptr);
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&maps.a);
    prefetch_tmap(&maps.b);
    if constexpr (Cfg::TF32) {
      prefetch_tmap(&maps.a_lo);
      prefetch_tmap(&maps.b_lo);
    }
    prefetch_tmap(&maps.c0);
    if constexpr (Cfg::NOUT > 1) prefetch_tmap(&maps.c1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      // COLSUM: the stage is free once the MMA commit AND the column-sum warp release it.
      mbar_init(&empty_bar[s], 1 + (colsum_live ? Cfg::COLSUM_WARPS : 0));
      if constexpr (Cfg::COLSUM) mbar_init(&ready_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], (Cfg::PAIR ? 2 : 1) * Cfg::EPI_WARPS * 32);  // both CTAs drain
    }
    if constexpr (Cfg::PRE_TMA)
      for (int w = 0; w < Cfg::EPI_WARPS; ++w) mbar_init(&pre_bar[w], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (Cfg::PAIR)
      tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);  // same warp id in both CTAs
    else
      tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (Cfg::PAIR)
    cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* const trace = args.trace;
  if (threadIdx.x == 0) {
    detail::trace_at(trace, 0);
    if (trace) trace[blockIdx.x * TRACE_STRIDE + TRACE_STRIDE - 1] = gridDim.x;  // lets readers walk the launches
  }
  // PDL: everything above (barrier init, TMEM alloc, descriptor prefetch)
  // overlapped the previous kernel's tail; global data is touched only after
  // it has completed. Then let the next kernel's prologue start.
  griddep_wait();
  if (args.ready_flag) {
    // every role reads the arriving shard (operands, FWD bias, the travelling
    // gradient's reduce-add and bias sums): each warp acquires the flag itself
    if ((threadIdx.x & 31) == 0) detail::wait_counter(args.ready_flag, 1u);
    __syncwarp();
  }
  // Only a running grid admits its successor: a grid still waiting for its
  // shard must not let the next launch on its stream take the SMs that the
  // other stream's kernels (the shard's producers' predecessors) need. (A
  // pass launch admits it once its producer is past the last step's wait; a
  // dW launch waiting for its travelling gradient once its epilogue has it.)
  if (!pass && !(Cfg::EPI == EPI_WGRAD && args.g_flag)) griddep_launch();
  if (threadIdx.x == 0) detail::trace_at(trace, 1);


  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
        if constexpr (Cfg::PAIR)
          tma_load_2d_pair(dst, m, bar, c0, c1);  // bytes counted on the leader's barrier
        else
          tma_load_2d(dst, m, bar, c0, c1);
      };
      // A box that lies entirely outside the tensor completes without
      // crediting bytes, so such boxes are skipped and the leader expects only
      // the bytes both CTAs actually request (their smem is never read into a
      // stored result: those rows / columns are clipped by the output maps).
      auto a_bytes = [&](int ma0, int M_) {
        int b = 0;
        if constexpr (Cfg::A_MN) {
          for (int c = 0; c < BM / Cfg::ATOM_MN; ++c)
            if (ma0 + c * Cfg::ATOM_MN < M_) b += BK * 128;
        } else {
          if (ma0 < M_) b = Cfg::A_BYTES;
        }
        return b * Cfg::NOPS;
      };
      auto b_bytes = [&](int nb0, int N_) {
        int b = 0;
        if constexpr (Cfg::B_MN) {
          for (int c = 0; c < Cfg::B_ROWS / Cfg::ATOM_MN; ++c)
            if (nb0 + c * Cfg::ATOM_MN < N_) b += BK * 128;
        } else {
          if (nb0 < N_) b = Cfg::B_BYTES;
        }
        return b * Cfg::NOPS;
      };
      int ready_step = 0;  // pass launch: steps whose shard is known to have landed
      bool admitted = false;
      for (int it = it_beg; it < it_end; it += it_step) {
        const Unit x = decode(it);
        const int mb = x.mb, nb = x.nb, kb0 = x.kb0, kb1 = x.kb1, uM = x.M, uN = x.N;
        const GemmMaps& mp = x.prob ? maps2 : maps;
        if (pass && Cfg::EPI != EPI_WGRAD && x.step > ready_step) {
          // (a pair's second shard came through the same comm stream after its first)
          const int last_step = args.pass_pair ? min(2 * x.step + 1, args.pass_steps - 1) : x.step;
          if (args.pass_ready) detail::wait_counter(args.pass_ready + last_step, 1u);
          ready_step = x.step;
        }
        if (pass && Cfg::EPI != EPI_WGRAD && x.step == pass_groups - 1 && !admitted) {  // the last shard landed
          griddep_launch();
          admitted = true;
        }
        // pass launch: the step's shard buffers and dY column blocks (per unit)
        const int first_step = args.pass_pair ? 2 * x.step : x.step;
        const bool dg_pass = pass && Cfg::EPI == EPI_DGRAD;
        const int a_koff0 = dg_pass ? args.pass_col[first_step] : 0;
        const int a_koff1 = dg_pass && x.seg_kb ? args.pass_col[first_step + 1] : 0;
        const int b_noff = (pass && Cfg::EPI == EPI_WGRAD) ? args.pass_col[x.step] : 0;  // dY column block
        const CUtensorMap* b_map0 = (pass && x.buf1) ? &maps2.b : &mp.b;
        if (x.prob && args.dep_count && !args.dep_on_k) {
          // problem 1 reads problem 0's output rows of this row block: wait
          // until every warp of every problem-0 tile of the block has landed
          // its stores, then order the async-proxy (TMA) reads after them.
          detail::wait_counter(args.dep_count + mb, args.dep_target);
        }
        int dep_rb = -1;  // dep_on_k: last row block waited for
        // this CTA's A rows and B columns (pair: its half of the 256 x BN tile)
        const int m0 = mb * Cfg::TILE_M + int(rank) * BM, n0 = nb * BN + int(rank) * Cfg::B_ROWS;
        int expect = a_bytes(mb * Cfg::TILE_M, uM) + b_bytes(nb * BN, uN);
        if constexpr (Cfg::PAIR) expect += a_bytes(mb * Cfg::TILE_M + BM, uM) + b_bytes(nb * BN + Cfg::B_ROWS, uN);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (x.prob && args.dep_on_k) {
            const int rb = (kb * BK) / 256;  // row block (256 rows) of the producing launch
            if (rb > dep_rb) {
              // wait for this row block, extend over the ones already complete
              // (up to the unit's last), then ONE proxy fence for all of them
              detail::wait_counter_nofence(args.dep_count + rb, args.dep_target);
              int r = rb;
              const int rb_last = ((kb1 - 1) * BK) / 256;
              while (r < rb_last && detail::ld_acquire(args.dep_count + r + 1) >= args.dep_target) ++r;
              asm volatile("fence.proxy.async.global;" ::: "memory");
              dep_rb = r;
            }
          }
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sA = stage_base + stage * Cfg::STAGE_BYTES;
          if (rank == 0) mbar_expect_tx(&full_bar[stage], uint32_t(expect));
          const bool seg2 = args.kseg_kb > 0 && kb >= args.kseg_kb;
          const GemmMaps& mk = seg2 ? maps2 : mp;
          const int k0 = (seg2 ? kb - args.kseg_kb : x.seg_kb && kb >= x.seg_kb ? kb - x.seg_kb : kb) * BK;
          // pass launch: this K block's shard buffer and dY column block
          const bool pseg2 = x.seg_kb && kb >= x.seg_kb;
          const CUtensorMap* b_map = pseg2 ? &maps2.b : b_map0;
          const int a_koff = pseg2 ? a_koff1 : a_koff0;
          for (int op = 0; op < Cfg::NOPS; ++op) {
            const CUtensorMap* ma = op ? &mk.a_lo : &mk.a;
            const CUtensorMap* mbm = op ? &mk.b_lo : (seg2 ? &mk.b : b_map);
            uint8_t* dA = sA + op * (Cfg::A_BYTES + Cfg::B_BYTES);
            uint8_t* dB = dA + Cfg::A_BYTES;
            if constexpr (Cfg::A_MN) {
#pragma unroll
              for (int c = 0; c < BM / Cfg::ATOM_MN; ++c)
                if (m0 + c * Cfg::ATOM_MN < uM)
                  load(dA + c * (BK * 128), ma, &full_bar[stage], m0 + c * Cfg::ATOM_MN, k0);
            } else {
              if (m0 < uM) load(dA, ma, &full_bar[stage], k0 + a_koff, m0);
            }
            if constexpr (Cfg::B_MN) {
#pragma unroll
              for (int c = 0; c < Cfg::B_ROWS / Cfg::ATOM_MN; ++c)
                if (n0 + c * Cfg::ATOM_MN < uN)
                  load(dB + c * (BK * 128), mbm, &full_bar[stage], n0 + c * Cfg::ATOM_MN + b_noff, k0);
            } else {
              if (n0 < uN) load(dB, mbm, &full_bar[stage], k0, n0);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair: leader CTA only) =====================
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int li = 0;
      for (int it = it_beg; it < it_end; it += it_step, ++li) {
        const Unit x = decode(it);
        const int kb0 = x.kb0, kb1 = x.kb1;
        const bool tr = trace && li < TRACE_UNITS;
        if (tr) detail::trace_at(trace, 2 + 6 * li);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        if (tr) detail::trace_at(trace, 3 + 6 * li);
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (tr && kb == kb0) detail::trace_at(trace, 4 + 6 * li);
          const uint32_t a_base = smem_u32(stage_base + stage * Cfg::STAGE_BYTES);
          const uint32_t b_base = a_base + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < Cfg::KSTEPS; ++kk) {
            // K-major: advance 32 B inside the 128B swizzle row.
            // MN-major: advance UMMA_K rows of 128 B (whole swizzle atoms).
            const uint32_t a_off = Cfg::A_MN ? kk * Cfg::UMMA_K * 128 : kk * 32;
            const uint32_t b_off = Cfg::B_MN ? kk * Cfg::UMMA_K * 128 : kk * 32;
            const uint32_t a_lbo = Cfg::A_MN ? BK * 128 : 16;
            const uint32_t b_lbo = Cfg::B_MN ? BK * 128 : 16;
            const uint64_t adesc = sdesc_sw128(a_base + a_off, a_lbo, 1024);
            const uint64_t bdesc = sdesc_sw128(b_base + b_off, b_lbo, 1024);
            const uint32_t accum = (kb != kb0) || kk != 0;
            if constexpr (Cfg::TF32) {
              constexpr uint32_t LO = Cfg::A_BYTES + Cfg::B_BYTES;
              const uint64_t adesc_lo = sdesc_sw128(a_base + LO + a_off, a_lbo, 1024);
              const uint64_t bdesc_lo = sdesc_sw128(b_base + LO + b_off, b_lbo, 1024);
              umma_tf32(d_tmem, adesc, bdesc, Cfg::IDESC, accum);
              umma_tf32(d_tmem, adesc, bdesc_lo, Cfg::IDESC, 1);
              umma_tf32(d_tmem, adesc_lo, bdesc, Cfg::IDESC, 1);
            } else if constexpr (Cfg::PAIR) {
              umma_f16_pair(d_tmem, adesc, bdesc, Cfg::IDESC, accum);
            } else {
              umma_f16(d_tmem, adesc, bdesc, Cfg::IDESC, accum);
            }
          }
          // free the stage in both CTAs / signal both CTAs' epilogues
          if constexpr (Cfg::PAIR)
            umma_commit_pair(&empty_bar[stage]);
          else
            umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (Cfg::PAIR)
          umma_commit_pair(&tfull_bar[acc]);
        else
          umma_commit(&tfull_bar[acc]);
        if (tr) detail::trace_at(trace, 5 + 6 * li);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp < 2 + Cfg::EPI_WARPS) {
    // ===================== Epilogue =====================
    const int ew = warp - 2;          // 0..EPI_WARPS-1
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int half = ew / 4;          // column interleave when EPI_WARPS == 8
    constexpr int NSPLIT = Cfg::EPI_WARPS / 4;
    uint8_t* stg0 = stg_base + ew * Cfg::STG_WARP;
    uint8_t* stg1 = stg0 + Cfg::STG_ONE;
    uint8_t* pre_w = pre_base + ew * Cfg::PRE_WARP;
    uint32_t pre_phase = 0;
    bool pending = false;
    bool g_ready = pass || args.g_flag == nullptr;  // WGRAD: travelling G landed (pass: step 0's is resident)
    const unsigned* gflag = pass ? nullptr : args.g_flag;  // WGRAD: the arrival flag of the unit's G
    unsigned wbuf = 0;  // dW staging buffer alternation
    int acc = 0;
    uint32_t acc_phase = 0;
    int li = 0;
    int e_step = 0;  // pass launch: step of the previous unit / whose shard is known landed
    for (int it = it_beg; it < it_end; it += it_step, ++li) {
      const bool tr = trace && li < TRACE_UNITS && ew == 0 && lane == 0;
      const Unit x_ = decode(it);
      const int t = x_.t, split = x_.split, mb = x_.mb, nb = x_.nb, uM = x_.M, uN = x_.N, uflags = x_.flags;
      const GemmMaps& mp = x_.prob ? maps2 : maps;
      const void* uaux = x_.prob ? args.aux2 : args.aux;
      if (pass && x_.step != e_step) {
        // Step boundary. DGRAD: this warp's bulk reductions of the previous
        // step are complete before the same tiles' next step reduces into /
        // reads the accumulator (fixed step order). FWD: the bias below lives
        // in the arriving shard. WGRAD: the step's G is a new arrival.
        if (Cfg::EPI == EPI_WGRAD) {
          gflag = args.pass_ready ? args.pass_ready + x_.step : nullptr;
          g_ready = gflag == nullptr;
        }
        if (lane == 0) {
          if (Cfg::EPI == EPI_DGRAD) {
            bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          if (Cfg::EPI == EPI_FWD && args.pass_ready) detail::wait_counter_nofence(args.pass_ready + x_.step, 1u);
        }
        __syncwarp();
        if (Cfg::EPI == EPI_DGRAD) pending = false;
        e_step = x_.step;
      }
      if (pass && Cfg::EPI == EPI_FWD) uaux = x_.buf1 ? args.aux2 : args.aux;
      const int col_off = (pass && Cfg::EPI == EPI_FWD) ? args.pass_col[x_.step] : 0;
      const bool last = uflags & EF_LAST;
      const bool first = uflags & EF_FIRST;
      const bool pre_tma = Cfg::PRE_TMA && last && (uflags & EF_GELU_BWD);
      const int wgroup = Cfg::EPI_WARPS * (Cfg::PAIR ? 2 : 1);  // epilogue warps per tile
      const int m0 = mb * Cfg::TILE_M + int(rank) * BM, n0 = nb * BN;  // this CTA's 128 rows
      const int row0 = m0 + q * 32;     // first row of this warp's 32-row slab
      const int row = row0 + lane;
      const bool row_ok = row < uM;
      if constexpr (Cfg::PRE_TMA) {
        // Stream this warp's pre chunks in while the tile's MMAs still run
        // (boxes entirely outside the tensor are skipped: they credit no bytes).
        if (pre_tma && lane == 0) {
          uint32_t bytes = 0;
          for (int k = 0; k < Cfg::PRE_CHUNKS; ++k)
            if (n0 + (half + k * NSPLIT) * 32 < uN && row0 < uM) bytes += 32 * 32 * Cfg::ELEM;
          mbar_expect_tx(&pre_bar[ew], bytes);
          for (int k = 0; k < Cfg::PRE_CHUNKS; ++k) {
            const int nc = n0 + (half + k * NSPLIT) * 32;
            if (nc < uN && row0 < uM)
              tma_load_2d(pre_w + k * 32 * 32 * Cfg::ELEM, &mp.c1, &pre_bar[ew], nc, row0);
          }
        }
      }
      float* bias_w = bias_base + ew * (Cfg::BIAS_WARP / 4);
      if constexpr (Cfg::EPI == EPI_FWD) {
        __syncwarp();  // every lane finished reading the previous tile's bias
        // lane i fetches column i of each of this warp's chunks (previous tile's
        // readers are done: the warp synchronised before releasing TMEM)
        for (int k = 0; k < Cfg::PRE_CHUNKS; ++k) {
          const int col = n0 + (half + k * NSPLIT) * 32 + lane;
          float bv = 0.f;
          if (col < uN && uaux) {  // no bias: projection blocks (RTPB_EPI_NO_BIAS)
            if constexpr (F32)
              bv = static_cast<const float*>(uaux)[col];
            else
              bv = __bfloat162float(static_cast<const __nv_bfloat16*>(uaux)[col]);
          }
          bias_w[k * 32 + lane] = bv;
        }
        __syncwarp();
      }
      // DGRAD last step: the warp's 32 x 32 fp32 accumulator chunk is loaded
      // coalesced (each instruction: 4 rows x 128 B, 4 L1 wavefronts instead
      // of 32 for one row per lane — the row-per-lane loads were bound by L1
      // wavefronts), two chunks ahead into two register buffers used
      // alternately, and transposed to row-per-lane through the staging
      // buffer (128 B swizzle, conflict-free).
      const bool acc_rd = Cfg::EPI == EPI_DGRAD && last && !first && row0 < uM;
      float4 acc_a[8], acc_b[8];
      auto load_acc = [&](int c, float4* d) {
        const int cc = c + (lane & 7) * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = row0 + i * 4 + (lane >> 3);
          d[i] = (r < uM && cc < uN)
                     ? *reinterpret_cast<const float4*>(args.acc + size_t(r) * args.ld_acc + cc)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      if constexpr (Cfg::EPI == EPI_DGRAD) {
        if (acc_rd && n0 + half * 32 < uN) load_acc(n0 + half * 32, acc_a);
        if (acc_rd && half + NSPLIT < BN / 32 && n0 + (half + NSPLIT) * 32 < uN)
          load_acc(n0 + (half + NSPLIT) * 32, acc_b);
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (tr) detail::trace_at(trace, 6 + 6 * li);
      if (pass && Cfg::EPI != EPI_WGRAD && args.pass_done && lane == 0) {
        // the tile's MMAs are done: its operand loads (and, FWD, this warp's
        // bias reads above) are complete — count in for the step's buffer
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(args.pass_done + x_.step) : "memory");
      }
      // FWD problem 1 split over K: partial splits go to the fp32 workspace,
      // in split order; the last split folds the workspace into its output.
      const bool split2 = Cfg::EPI == EPI_FWD && x_.prob == 1 && splits2 > 1 && !x_.whole;
      const bool part2 = split2 && split < splits2 - 1;
      const bool fin2 = split2 && split == splits2 - 1;
      if (split2 && split > 0) {
        if (lane == 0) detail::wait_counter(args.split_flags2 + t, unsigned(split * wgroup));
        __syncwarp();
      }
      // dW split over K (per problem): its own counters
      unsigned* const wflags = x_.prob ? args.split_flags2 : args.split_flags;
      const int wsplits = x_.prob ? splits2 : splits;
      const bool wpar = Cfg::EPI == EPI_WGRAD && args.wpar && wsplits > 1;
      const int wprows = x_.prob ? args.wpart_rows2 : args.wpart_rows;
      // ordered split-K chain counter of the tile (a pass launch: one per
      // step among the tile's 16 slots, so steps never share a chain)
      unsigned* const chain_ctr = pass ? wflags + t * 16 + (x_.step & 15) : wflags + t;
      if constexpr (Cfg::EPI == EPI_WGRAD) {
        // the travelling G must have landed before this warp's first update
        // of it (first && split 0 overwrite it: G is known zero, no wait;
        // split partials go to the workspace: their folds wait below)
        if (!g_ready && !wpar && !(first && split == 0)) {
          if (lane == 0) detail::wait_counter(gflag, 1u);
          __syncwarp();
          g_ready = true;
          if (ew == 0 && lane == 0 && (!pass || x_.step == pass_groups - 1)) griddep_launch();  // G landed: admit the successor
        }
        if (split > 0 && !wpar) {
          // ordered split-K: wait until every warp of split-1 has landed its sums
          if (lane == 0) detail::wait_counter(chain_ctr, unsigned(split * wgroup));
          __syncwarp();
        }
      }
      if constexpr (Cfg::PRE_TMA) {
        if (pre_tma) {
          mbar_wait(&pre_bar[ew], pre_phase);
          pre_phase ^= 1;
        }
      }
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int ch = half; ch < BN / 32; ch += NSPLIT) {
        const int nc = n0 + ch * 32;
        if (nc >= uN) break;  // warp-uniform
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + ch * 32, v);
        tmem_ld_wait();
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(v[e]);
        // staging buffers free again (previous chunk's bulk stores read them);
        // dW alternates two buffers and waits only for the older group
        uint8_t* wstg = stg0;
        if constexpr (Cfg::EPI == EPI_WGRAD && Cfg::STG_BUFS == 2) {
          wstg = (wbuf & 1) ? stg1 : stg0;
          ++wbuf;
        }
        if (pending) {
          if (lane == 0) {
            if constexpr (Cfg::EPI == EPI_WGRAD && Cfg::STG_BUFS == 2)
              bulk_wait_read1();
            else
              bulk_wait_read0();
          }
          __syncwarp();
        }
        if constexpr (Cfg::EPI == EPI_FWD) {
          if (part2) {
            detail::stage_row<true>(stg0, lane, x);  // fp32 partial (stg0 + stg1: 4 KB)
          } else {
            if (fin2 && row_ok) {
#pragma unroll
              for (int g = 0; g < 4; ++g)
                if (nc + g * 8 < uN) {
                  const float4* p = reinterpret_cast<const float4*>(args.acc2 + row * args.ld_acc2 + nc + g * 8);
                  const float4 a = __ldcg(p), b = __ldcg(p + 1);
                  x[g * 8 + 0] += a.x; x[g * 8 + 1] += a.y; x[g * 8 + 2] += a.z; x[g * 8 + 3] += a.w;
                  x[g * 8 + 4] += b.x; x[g * 8 + 5] += b.y; x[g * 8 + 6] += b.z; x[g * 8 + 7] += b.w;
                }
            }
            const float4* bsm = reinterpret_cast<const float4*>(bias_w + ((ch - half) / NSPLIT) * 32);
#pragma unroll
            for (int g = 0; g < 8; ++g) {  // broadcast smem reads
              const float4 b4 = bsm[g];
              x[4 * g] += b4.x;
              x[4 * g + 1] += b4.y;
              x[4 * g + 2] += b4.z;
              x[4 * g + 3] += b4.w;
            }
            if (uflags & EF_STORE_PRE) detail::stage_row<F32>(stg0, lane, x);
            if (uflags & EF_GELU) {
              if (!F32 && (uflags & EF_EXACT_GELU)) {  // warp-uniform: one loop or the other
#pragma unroll
                for (int e = 0; e < 32; ++e) x[e] = detail::gelu_f<true>(x[e]);
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) x[e] = detail::gelu_f<F32>(x[e]);
              }
              detail::stage_row<F32>(stg1, lane, x);
            }
          }
        } else if constexpr (Cfg::EPI == EPI_DGRAD) {
          if (acc_rd) {
            // consume this chunk's buffer (transpose through stg0, free: the
            // previous chunk's store has read it), refill it two chunks ahead
            const int nn = nc + 2 * NSPLIT * 32;
            const bool more = ch + 2 * NSPLIT < BN / 32 && nn < uN;
            auto put = [&](const float4* d) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int r = i * 4 + (lane >> 3), k = lane & 7;
                *reinterpret_cast<float4*>(stg0 + r * 128 + ((k ^ (r & 7)) * 16)) = d[i];
              }
            };
            if ((((ch - half) / NSPLIT) & 1) == 0) {
              put(acc_a);
              if (more) load_acc(nn, acc_a);
            } else {
              put(acc_b);
              if (more) load_acc(nn, acc_b);
            }
            __syncwarp();
            float av[32];
            detail::unstage_row<true>(stg0, lane, av);
#pragma unroll
            for (int e = 0; e < 32; ++e) x[e] += av[e];
            __syncwarp();  // every lane has read stg0 before the output is staged over it
          }
          if (pre_tma) {
            // pre chunk staged by TMA in the same swizzled 32 x 32 layout as the outputs
            const uint8_t* pc = pre_w + ((ch - half) / NSPLIT) * 32 * 32 * Cfg::ELEM;
            float pre[32];
            detail::unstage_row<F32>(pc, lane, pre);
            if (!F32 && (uflags & EF_EXACT_GELU)) {
#pragma unroll
              for (int e = 0; e < 32; ++e) x[e] *= detail::gelu_grad_f<true>(pre[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) x[e] *= detail::gelu_grad_f<F32>(pre[e]);
            }
          } else if (last && (uflags & EF_GELU_BWD) && row_ok) {
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (nc + g * 8 < uN) {
                float pre[8];
                detail::load8<F32>(uaux, row * args.ld_aux + nc + g * 8, pre);
                if (!F32 && (uflags & EF_EXACT_GELU)) {
#pragma unroll
                  for (int e = 0; e < 8; ++e) x[g * 8 + e] *= detail::gelu_grad_f<true>(pre[e]);
                } else {
#pragma unroll
                  for (int e = 0; e < 8; ++e) x[g * 8 + e] *= detail::gelu_grad_f<F32>(pre[e]);
                }
              }
          }
          if (last)
            detail::stage_row<F32>(stg0, lane, x);
          else
            detail::stage_row<true>(stg0, lane, x);
        } else {
          detail::stage_row<true>(wstg, lane, x);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (Cfg::EPI == EPI_FWD) {
            if (part2) {
              if (split == 0)
                tma_store_2d(&mp.c1, stg0, nc, row0);  // workspace = partial 0
              else
                tma_reduce_add_2d(&mp.c1, stg0, nc, row0);  // workspace += partial s
            } else {
              if (uflags & EF_STORE_PRE) tma_store_2d(&mp.c0, stg0, col_off + nc, row0);
              if (uflags & EF_GELU) tma_store_2d(&mp.c1, stg1, col_off + nc, row0);
            }
          } else if constexpr (Cfg::EPI == EPI_DGRAD) {
            if (pass && last)
              tma_store_2d(&maps2.c0, stg0, nc, row0);  // pass launch: dX map beside the accumulator's
            else if (last || first)
              tma_store_2d(&mp.c0, stg0, nc, row0);  // dX (dtype) or first partial (fp32)
            else
              tma_reduce_add_2d(&mp.c0, stg0, nc, row0);  // acc += partial, in L2
          } else {
            if (wpar)
              tma_store_2d(&mp.c1, wstg, nc, split * wprows + row0);  // this split's partial
            else if (first && split == 0)
              tma_store_2d(&mp.c0, wstg, nc, row0);  // G known zero: G = dW tile (split 0 lands first)
            else
              tma_reduce_add_2d(&mp.c0, wstg, nc, row0);  // travelling G += dW tile
          }
          bulk_commit();
        }
        pending = true;
      }
      if (split2) {
        // publish (tile, split) done; the last arrival of the last split re-zeroes
        if (lane == 0) {
          bulk_wait0();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          const unsigned old = atomicAdd(args.split_flags2 + t, 1u);
          if (old + 1 == unsigned(splits2 * wgroup)) args.split_flags2[t] = 0u;
        }
        __syncwarp();
        pending = false;
      }
      if constexpr (Cfg::EPI == EPI_WGRAD) {
        if (wpar && args.wpar == 2) {
          // All splits of the launch are resident (units <= slots): every
          // split stores its partial, waits until the region's S partials are
          // in, then folds its own slice of the region's 32 rows (partials in
          // split order, then + G_in) with plain stores — no chain of
          // serialised epilogues. Deterministic: one owner per row.
          const int slot = int(rank) * Cfg::EPI_WARPS + ew;
          unsigned* cnt = wflags + t * wgroup + slot;
          if (lane == 0) {
            bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            atomicAdd(cnt, 1u);
            detail::wait_counter_nofence(cnt, unsigned(wsplits));
            __threadfence();
          }
          __syncwarp();
          pending = false;
          if (!g_ready && !first) {  // the fold reads G
            if (lane == 0) detail::wait_counter_nofence(gflag, 1u);
            __syncwarp();
            g_ready = true;
            if (ew == 0 && lane == 0 && (!pass || x_.step == pass_groups - 1)) griddep_launch();  // G landed: admit the successor
          }
          const float* part = x_.prob ? args.wpart2 : args.wpart;
          const int r_lo = (32 * split) / wsplits, r_hi = (32 * (split + 1)) / wsplits;
          float* gout = const_cast<float*>(static_cast<const float*>(x_.prob ? args.gout2 : args.gout));
          // Each lane takes one column of every 32-column chunk of the slice's
          // rows, so every load and store is a coalesced 128-byte row segment
          // (a row per lane costs 32 L1 wavefronts per instruction). All S
          // partials of an element are loaded before the sum, added in split
          // order, then G: the same order, and bits, as the chained folds.
          // Every load of a group (RPI rows x all of the warp's chunks x the S
          // partials, and G) is issued before the first sum, so the fold costs
          // one L2 round trip per group instead of two per (row, chunk).
          constexpr int CH = BN / 32 / NSPLIT;      // chunks of this warp
          constexpr int RPI = CH <= 2 ? 2 : 1;      // rows per group
          for (int r = r_lo; r < r_hi; r += RPI) {
            float tv[RPI][CH][8], gv[RPI][CH];
#pragma unroll
            for (int i = 0; i < RPI; ++i)
#pragma unroll
              for (int c = 0; c < CH; ++c) {
                const int grow = row0 + r + i;
                const int col = n0 + (half + c * NSPLIT) * 32 + lane;
                const bool ok = r + i < r_hi && grow < uM && col < uN;
#pragma unroll
                for (int sp = 0; sp < 8; ++sp)
                  tv[i][c][sp] = ok && sp < wsplits ? __ldcg(part + (size_t(sp) * wprows + grow) * uN + col) : 0.f;
                gv[i][c] = ok && !first ? __ldcg(gout + size_t(grow) * uN + col) : 0.f;
              }
#pragma unroll
            for (int i = 0; i < RPI; ++i)
#pragma unroll
              for (int c = 0; c < CH; ++c) {
                const int grow = row0 + r + i;
                const int col = n0 + (half + c * NSPLIT) * 32 + lane;
                if (r + i < r_hi && grow < uM && col < uN) {
                  float a = 0.f;
#pragma unroll
                  for (int sp = 0; sp < 8; ++sp)
                    if (sp < wsplits) a += tv[i][c][sp];
                  if (!first) a = gv[i][c] + a;
                  gout[size_t(grow) * uN + col] = a;
                }
              }
          }
          __syncwarp();
          if (lane == 0) {  // count out; the last split out re-zeroes the region counter
            __threadfence();
            if (atomicAdd(cnt, 1u) + 1 == unsigned(2 * wsplits)) *cnt = 0u;
          }
        } else if (wpar) {
          // count in on this warp's region; the warp completing it folds the
          // partials (split order) into G
          const int slot = int(rank) * Cfg::EPI_WARPS + ew;
          unsigned* cnt = wflags + t * wgroup + slot;
          unsigned last = 0;
          if (lane == 0) {
            bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            last = atomicAdd(cnt, 1u) + 1 == unsigned(wsplits);
            if (last) __threadfence();
          }
          last = __shfl_sync(0xffffffffu, last, 0);
          pending = false;
          if (last && !g_ready && !first) {  // the fold reduce-adds into G
            if (lane == 0) detail::wait_counter(gflag, 1u);
            __syncwarp();
            g_ready = true;
            if (ew == 0 && lane == 0 && (!pass || x_.step == pass_groups - 1)) griddep_launch();  // G landed: admit the successor
          }
          if (last) {
            const float* part = x_.prob ? args.wpart2 : args.wpart;
#pragma unroll 1
            for (int ch = half; ch < BN / 32; ch += NSPLIT) {
              const int nc = n0 + ch * 32;
              if (nc >= uN) break;
              float x[32];
#pragma unroll
              for (int e = 0; e < 32; ++e) x[e] = 0.f;
              if (row_ok) {
                for (int sp = 0; sp < wsplits; ++sp) {
                  const float* src = part + (size_t(sp) * wprows + row) * uN + nc;
#pragma unroll
                  for (int g = 0; g < 4; ++g)
                    if (nc + g * 8 < uN) {
                      const float4 a = __ldcg(reinterpret_cast<const float4*>(src + g * 8));
                      const float4 b = __ldcg(reinterpret_cast<const float4*>(src + g * 8) + 1);
                      x[g * 8 + 0] += a.x; x[g * 8 + 1] += a.y; x[g * 8 + 2] += a.z; x[g * 8 + 3] += a.w;
                      x[g * 8 + 4] += b.x; x[g * 8 + 5] += b.y; x[g * 8 + 6] += b.z; x[g * 8 + 7] += b.w;
                    }
                }
              }
              if (pending) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              detail::stage_row<true>(stg0, lane, x);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                if (first)
                  tma_store_2d(&mp.c0, stg0, nc, row0);
                else
                  tma_reduce_add_2d(&mp.c0, stg0, nc, row0);
                bulk_commit();
              }
              pending = true;
            }
            if (lane == 0) *cnt = 0u;  // every split of this region has counted in
          }
        } else if (wsplits > 1) {
          // publish: this warp's reduce-adds for (tile, split) are performed
          if (lane == 0) {
            bulk_wait0();
            __threadfence();
            const unsigned old = atomicAdd(chain_ctr, 1u);
            if (old + 1 == unsigned(wsplits * wgroup)) *chain_ctr = 0u;  // last arrival re-zeroes
          }
          __syncwarp();
          pending = false;
        }
      }
      if constexpr (Cfg::EPI == EPI_WGRAD) {
        if (pass) {
          if (t == 0 && split == 0 && ew == 0 && rank == 0 && args.pass_db) {
            // G's bias part: + this step's dY column sums, once G(s) is here
            if (!g_ready && !first) {
              if (lane == 0) detail::wait_counter_nofence(gflag, 1u);
              __syncwarp();
              g_ready = true;
            }
            const float* db = args.pass_db + args.pass_col[x_.step];
            for (int c = lane; c < uN; c += 32) args.pass_gbias[c] = (first ? 0.f : args.pass_gbias[c]) + db[c];
            __syncwarp();
          }
          // count in once this warp's updates of G have landed: the comm
          // stream sends G on when the step's count-ins are complete
          if (lane == 0) {
            bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            if (args.pass_done)
              asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(args.pass_done + x_.step) : "memory");
          }
          __syncwarp();
          pending = false;
        }
      }
      if constexpr (Cfg::PRE_TMA) __syncwarp();  // all lanes done with the pre chunks
      if (tr) detail::trace_at(trace, 7 + 6 * li);
      tc_fence_before();
      if constexpr (Cfg::PAIR)
        mbar_arrive_cluster(&tempty_bar[acc], 0);  // the leader's MMA reuses both halves
      else
        mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (args.dep_count && !args.dep_on_k && x_.prob == 0) {
        // publish: this warp's stores of the tile are complete (problem 1
        // reads them as its A operand), after the accumulator was released.
        // (A dep_on_k launch only consumes another launch's counters.)
        if (lane == 0) {
          bulk_wait0();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          atomicAdd(args.dep_count + mb, 1u);
        }
        __syncwarp();
        pending = false;
      }
    }
    if (lane == 0) bulk_wait0();
    __syncwarp();
  } else if constexpr (Cfg::COLSUM) {
    // ============ Bias gradient: column sums of the staged dY (B) tiles ============
    // B stage layout (MN-major, SWIZZLE_128B): chunk c holds columns
    // [64c, 64c+64) as BK rows of 128 B; 16-byte piece j of row k sits at
    // piece j ^ (k & 7). Lane: 8 columns (one piece) of every RPI-th row.
    // Every tile row block mb sees the same dY columns, so the work is spread:
    // unit (mb, nb, split) sums only the k-blocks with kb % num_m == mb, writes
    // that partial to its own workspace row, and the last of the num_m * splits
    // contributors of a column group adds them up in a fixed order
    // (deterministic, no waiting).
    constexpr int NCH = Cfg::B_ROWS / 64;   // 64-column chunks per CTA (1 or 2)
    constexpr int LPR = 8 * NCH;            // lanes per row
    constexpr int RPI = 32 / LPR;           // rows per warp-wide step
    constexpr int ROWS = BK / Cfg::COLSUM_WARPS;
    const int cw = warp - 2 - Cfg::EPI_WARPS;  // 0: publisher, 1: helper
    const int chunk = (lane % LPR) / 8, piece = lane & 7, rsub = lane / LPR;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = it_beg; colsum_live && it < it_end; it += it_step) {
      const Unit x_ = decode(it);
      const int split = x_.split, mb = x_.mb, nb = x_.nb, kb0 = x_.kb0, kb1 = x_.kb1, uN = x_.N;
      const bool first = x_.flags & EF_FIRST;
      const int unum_m = x_.prob ? num_m2 : num_m;
      const int contributors = unum_m * (x_.prob ? splits2 : splits);
      const float* ugb_in = x_.prob ? args.gbias_in2 : args.gbias_in;
      float* ugb_out = x_.prob ? args.gbias_out2 : args.gbias_out;
      float* upart = x_.prob ? args.bias_part2 : args.bias_part;
      unsigned* utick = x_.prob ? args.bias_tick2 : args.bias_tick;
      const bool colsum_on = Cfg::COLSUM && ugb_out != nullptr;
      float sum[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) sum[e] = 0.f;
      for (int kb = kb0; kb < kb1; ++kb) {
        // Leader: the stage's full barrier counts both CTAs' bytes; its first
        // column-sum warp forwards the event to the peer (off the MMA thread).
        if (rank == 0) {
          mbar_wait(&full_bar[stage], phase);
          // (default .release.cta remote arrive: a cluster-scope release
          // compiles to MEMBAR.ALL.GPU and stalled the pipeline ~1 us / stage)
          if (cw == 0 && lane == 0) mbar_arrive_cluster(&ready_bar[stage], 1);
        } else {
          mbar_wait(&ready_bar[stage], phase);
        }
        if (colsum_on && kb % unum_m == mb) {
          const uint8_t* sB = stage_base + stage * Cfg::STAGE_BYTES + Cfg::A_BYTES + chunk * (BK * 128);
#pragma unroll 4
          for (int i = 0; i < ROWS / RPI; ++i) {
            const int k = cw * ROWS + i * RPI + rsub;  // rows past K were zero-filled by TMA
            const uint4 v = *reinterpret_cast<const uint4*>(sB + k * 128 + ((piece ^ (k & 7)) << 4));
            detail::acc_bf16x2(sum[0], sum[1], v.x);
            detail::acc_bf16x2(sum[2], sum[3], v.y);
            detail::acc_bf16x2(sum[4], sum[5], v.z);
            detail::acc_bf16x2(sum[6], sum[7], v.w);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!colsum_on) continue;
      // fold the row subsets: lanes 0..LPR-1 then hold columns lane*8 .. lane*8+7
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e) sum[e] += __shfl_xor_sync(0xffffffffu, sum[e], o);
      float4* cs = reinterpret_cast<float4*>(csum_base) + lane * 2;
      if (cw == 1 && lane < LPR) {
        cs[0] = make_float4(sum[0], sum[1], sum[2], sum[3]);
        cs[1] = make_float4(sum[4], sum[5], sum[6], sum[7]);
      }
      named_bar_sync(1, 64);
      if (cw == 0) {
        const int cg = nb * 2 + int(rank);                 // this CTA's column group
        const int c0 = cg * Cfg::B_ROWS + lane * 8;
        float* part = upart + size_t(split * unum_m + mb) * uN;
        if (lane < LPR) {
          const float4 a = cs[0], b = cs[1];
          sum[0] += a.x; sum[1] += a.y; sum[2] += a.z; sum[3] += a.w;
          sum[4] += b.x; sum[5] += b.y; sum[6] += b.z; sum[7] += b.w;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c0 + e < uN) part[c0 + e] = sum[e];
        }
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
          __threadfence();
          const unsigned old = atomicAdd(utick + cg, 1u);
          last = old + 1 == unsigned(contributors);
          if (last) {
            utick[cg] = 0u;  // self-resetting for the next launch
            __threadfence();
          }
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        __syncwarp();
        if (last) {
          // Every contributor's partial is visible. All 32 lanes help: lane
          // group g = lane / LPR sums contributors r = g, g + G, ... in
          // ascending order (loads of 4 contributors in flight at a time,
          // float4-wide), then the G group sums are added in group order:
          // a fixed order, so the result is bitwise reproducible. (A serial
          // per-column loop here held the stage release of this CTA's next
          // unit for tens of microseconds.)
          constexpr int G = 32 / LPR;
          const int grp = lane / LPR, cl = cg * Cfg::B_ROWS + (lane % LPR) * 8;
          float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
          if (cl < uN) {
            const float* base = upart + cl;
            int r = grp;
            for (; r + 3 * G < contributors; r += 4 * G) {
              float4 v[8];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4* p = reinterpret_cast<const float4*>(base + size_t(r + q * G) * uN);
                v[2 * q] = __ldcg(p);
                v[2 * q + 1] = __ldcg(p + 1);
              }
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                s0.x += v[2 * q].x; s0.y += v[2 * q].y; s0.z += v[2 * q].z; s0.w += v[2 * q].w;
                s1.x += v[2 * q + 1].x; s1.y += v[2 * q + 1].y; s1.z += v[2 * q + 1].z; s1.w += v[2 * q + 1].w;
              }
            }
            for (; r < contributors; r += G) {
              const float4* p = reinterpret_cast<const float4*>(base + size_t(r) * uN);
              const float4 a = __ldcg(p), b = __ldcg(p + 1);
              s0.x += a.x; s0.y += a.y; s0.z += a.z; s0.w += a.w;
              s1.x += b.x; s1.y += b.y; s1.z += b.z; s1.w += b.w;
            }
          }
          const float4 t0 = s0, t1 = s1;  // group sums, read unmodified by the shuffles
#pragma unroll
          for (int g = 1; g < G; ++g) {
            const int src = (lane + g * LPR) & 31;
            s0.x += __shfl_sync(0xffffffffu, t0.x, src); s0.y += __shfl_sync(0xffffffffu, t0.y, src);
            s0.z += __shfl_sync(0xffffffffu, t0.z, src); s0.w += __shfl_sync(0xffffffffu, t0.w, src);
            s1.x += __shfl_sync(0xffffffffu, t1.x, src); s1.y += __shfl_sync(0xffffffffu, t1.y, src);
            s1.z += __shfl_sync(0xffffffffu, t1.z, src); s1.w += __shfl_sync(0xffffffffu, t1.w, src);
          }
          if (!first && args.g_flag) {  // G's bias part is read below
            if (lane == 0) detail::wait_counter_nofence(args.g_flag, 1u);
            __syncwarp();
          }
          if (lane < LPR && cl < uN) {
            float4* o = reinterpret_cast<float4*>(ugb_out + cl);
            if (!first) {
              const float4* gi = reinterpret_cast<const float4*>(ugb_in + cl);
              const float4 a = __ldcg(gi), b = __ldcg(gi + 1);
              s0 = make_float4(a.x + s0.x, a.y + s0.y, a.z + s0.z, a.w + s0.w);
              s1 = make_float4(b.x + s1.x, b.y + s1.y, b.z + s1.z, b.w + s1.w);
            }
            o[0] = s0;
            o[1] = s1;
          }
        }
      }
      named_bar_sync(1, 64);  // partial buffer free for the next unit
    }
  }

  tc_fence_before();
  if constexpr (Cfg::PAIR)
    cluster_sync();  // both CTAs done with TMEM / remote barriers before release
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (Cfg::PAIR)
      tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
  if (args.flag_reset && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(args.flag_reset_ctr, 1u) == gridDim.x - 1) {
      for (int i = 0; i < args.flag_reset_count; ++i) args.flag_reset[i] = 0u;
      // pass launch: every count-in happened before this CTA's exit, and the
      // comm stream's waits on them were satisfied before the pass's last
      // arrival flag it raised (which every CTA passed)
      if (args.pass_done)
        for (int i = 0; i < args.pass_steps; ++i) args.pass_done[i] = 0u;
      *args.flag_reset_ctr = 0u;
      __threadfence();
    }
  }
  if (args.dep_count && threadIdx.x == 0) {
    // every thread of this CTA is past its last dependency read: the last CTA
    // out re-zeroes the row-block counters for the next launch
    __threadfence();
    if (atomicAdd(args.done_ctas, 1u) == (args.done_target ? args.done_target : gridDim.x) - 1) {
      for (int r = 0; r < args.dep_rows; ++r) args.dep_count[r] = 0u;
      *args.done_ctas = 0u;
      __threadfence();
    }
  }
}

}  // namespace rtpb
