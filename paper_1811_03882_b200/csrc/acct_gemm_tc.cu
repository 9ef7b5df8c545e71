// gemm_nn on the 5th-generation tensor cores, FP32-accurate via 3xTF32.
//
//   C[M][N] = beta*C + alpha * A[M][K] . B[K][N]  (+ bias[row]) (leaky)
//
// A (the layer's weights) is row-major, K contiguous -> a "K-major" UMMA
// operand; B (im2col columns / activations) is row-major, N contiguous -> an
// "MN-major" operand (legal for kind::tf32 only in the SWIZZLE_128B_BASE32B
// shared-memory layout, TMA swizzle 128B_ATOM_32B).  Each operand x is split
// exactly into x_hi = x with the low 13 mantissa bits cleared (a TF32 value)
// and x_lo = x - x_hi (exact in FP32; truncated to TF32 by the MMA), and the
// tile accumulates  X_hi.Y_hi + X_hi.Y_lo + X_lo.Y_hi  in TMEM (FP32), which
// keeps the product within ~2^-20 relative of FP32 -- the accuracy contract
// of darknet's FP32 gemm_nn (tests: 1e-4 scale-relative, 1e-5 normwise).
// tcgen05 kind::tf32 truncates FP32 operands itself (measured bit-identical,
// tests/test_gpu_kernels.py::test_tf32_operand_truncation), so the raw value
// stays in shared memory as x_hi and only x_lo is written.
//
// Two tile orientations (MMA M is always 128 rows = TMEM lanes):
//   normal  X = 128 weight rows (K-major), Y = TN in {128, 192} columns of B
//           (MN-major): the wide-M layers; TN = 192 covers the 13x13 layers
//           (N = 169) with one N tile.
//   swap    X = 128 columns of B (MN-major), Y = TN in {16, 32, 64} weight
//           rows (K-major): C^T = B^T A^T for the narrow-M layers (M = 16, 32,
//           64), so no MMA rows are wasted; TMEM lanes are output columns and
//           epilogue stores coalesce as they come.
//
// Persistent, warp-specialized CTA (one per SM, 10 warps) looping over work
// units (tile x K-split) round-robin:
//   warp 0      TMA producer (one elected lane): a continuous `stages`-deep
//               ring of k-blocks that runs across unit boundaries
//   warp 1      TMEM allocator + MMA issuer (one elected lane); two TMEM
//               accumulators so unit j+1 accumulates while unit j drains
//   warps 2..5  hi/lo split of each landed stage (lo to its own buffer;
//               generic -> async proxy fence before the release)
//   warps 6..9  epilogue: tcgen05.ld -> registers -> (normal tiles: smem
//               transpose) -> coalesced 128-B row stores with beta*C, bias and
//               leaky fused; under split-K, raw FP32 partials to an L2-resident
//               workspace summed in split order by a grid-wide kernel
//               (deterministic run to run)
// Barriers: per stage full (TMA bytes landed) / conv (split done, 4 warp
// arrivals) / empty (tcgen05.commit after the stage's MMAs); per accumulator
// acc_full (commit after a unit's last k-block) / acc_empty (4 epilogue warps).
// BK is the k depth of one stage: 32 (128-B K-major rows, SWIZZLE_128B) or 16
// (64-B rows, SWIZZLE_64B) so the 80-KB/stage TN=192 tile still gets a deep
// ring.

#include <cuda.h>

#include <cfloat>

#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "acct_common.cuh"
#include "acct_tc.cuh"

namespace acct {
namespace {

// warps: 0 TMA, 1 MMA, 2-5 split, 6-9 and 10-13 two epilogue groups that take
// alternate work units (one group's drain overlaps the other's)
constexpr int EPI_GROUPS = 2;
constexpr int THREADS = 32 * (6 + 4 * EPI_GROUPS);
constexpr int STAGING_BYTES = EPI_GROUPS * 4 * 32 * 33 * 4;  // normal-tile epilogue transpose

// bit 0: store x_hi explicitly (default 0: leave the raw FP32 value in place --
// tcgen05 kind::tf32 reads only the TF32 bits of each operand).  Bits 1-3
// skip the split / MMA / epilogue work (results wrong): honoured only by the
// -DACCT_PROFILING build of tools/gemm_bench.py (ACCT_SKIP), compiled out of
// the product library.
int g_write_hi = 0;
// normal-orientation tile override (0 = cost model; tests/tools only):
// 1 = 128x192 (A in TMEM), 2 = 128x128 BK16, 3 = 128x128 BK32, 4 = 128x256,
// 5/6/7 = CTA pair 256x192 / 256x256 / 256x128.  Initialised from ACCT_TC_TILE.
std::atomic<int> g_force_tile{-1};
int forced_tile() {
  int v = g_force_tile.load(std::memory_order_relaxed);
  if (v < 0) {
    const char *e = getenv("ACCT_TC_TILE");
    v = e ? atoi(e) : 0;
    g_force_tile.store(v, std::memory_order_relaxed);
  }
  return v;
}
// bit 4: event trace of CTA 0's first kTrace stages (clock64 per role), read
// back with acct_tc_trace -- pipeline analysis only (tools/tc_trace.py)
constexpr int kTrace = 512;
__device__ long long g_trace[12][kTrace];
// bits 8-15 of the same word: L2 prefetch distance in k-blocks (ACCT_TC_PF,
// default 0: measured slower for every net shape -- the ring is not HBM-latency bound)
int prefetch_distance() {
  static const int pf = [] {
    const char *e = getenv("ACCT_TC_PF");
    int v = e ? atoi(e) : 0;
    return v < 0 ? 0 : (v > 255 ? 255 : v);
  }();
  return pf;
}

// AT: the weight tile (MMA operand A) goes to TMEM -- the split warps read it
// from shared memory once and store hi and lo with tcgen05.st, so the MMAs
// read only B from shared memory.  Shared-memory bandwidth is the binding
// limit of 3xTF32 on one SM (per 16-deep k-block: TMA 20 KB + split 40 KB +
// MMA operand reads 60 KB vs 576 MMA cycles x 128 B/cycle), and AT cuts it
// from 120 KB to 88 KB per k-block.
template <int TN, int BK, bool AT>
struct Cfg {
  static constexpr int X_TILE = 128 * BK * 4;
  static constexpr int Y_TILE = TN * BK * 4;
  // raw(hi) + lo of both operands; with AT the A lo lives in TMEM
  static constexpr int STAGE_BYTES = (AT ? 1 : 2) * X_TILE + 2 * Y_TILE;
  static constexpr int BUDGET = 220 * 1024 - STAGING_BYTES - 512 - 1024;
  // TMEM accumulator ring: 4 buffers when they fit in 512 columns, else 2
  static constexpr int NACC = 4 * TN <= 512 ? 4 : 2;
  static constexpr int SMEM_STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  // with AT each stage also holds 2 x BK TMEM columns (A hi, A lo)
  static constexpr int TMEM_STAGES = AT ? (512 - NACC * TN) / (2 * BK) : 8;
  static constexpr int STAGES = SMEM_STAGES < TMEM_STAGES ? SMEM_STAGES : TMEM_STAGES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 512 + 1024;
  static constexpr int A_COL0 = NACC * TN;                    // first A-stage TMEM column
  static constexpr int USED_COLS = NACC * TN + (AT ? STAGES * 2 * BK : 0);
  static constexpr uint32_t TMEM_COLS = USED_COLS <= 32 ? 32 : USED_COLS <= 64 ? 64
                                       : USED_COLS <= 128 ? 128 : USED_COLS <= 256 ? 256 : 512;
  // K-major operand (rows x BK fp32)
  static constexpr uint32_t KROW = BK * 4;                    // 128 or 64 bytes
  static constexpr uint32_t K_LAYOUT = BK == 32 ? ptx::kLayoutSW128 : 4u /*SWIZZLE_64B*/;
  static constexpr uint32_t K_SBO = 8 * KROW;                 // 8-row swizzle atom
  // MN-major operand (BK rows x 32-column chunks)
  static constexpr uint32_t MN_CHUNK = BK * 128;              // LBO between 32-col chunks
  static_assert(STAGES >= 2, "tile does not fit shared memory");
  static_assert(USED_COLS <= 512, "TMEM overflow");
};

template <int TN, bool SWAP, int BK>
struct Pick {
  static constexpr bool AT = (!SWAP && TN == 192 && BK == 16) || (SWAP && BK == 32);
  using G = Cfg<TN, BK, AT>;
};

__device__ __forceinline__ float4 split_lo(float4 v, float4 &hi) {
  hi.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
  hi.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
  hi.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
  hi.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
  return make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
}

// epilogue arithmetic without the activation (applied per block of values
// with acct_leaky_block, one guard vote per block)
__device__ __forceinline__ float finish_lin(float acc, float alpha, float beta, float c,
                                            const float *bias, float bias_v) {
  float v = alpha * acc;
  if (beta != 0.0f) v = beta * c + v;
  if (bias) v += bias_v;
  return v;
}

struct Unit {
  int n0, m0, split, kb0, nkb;
};

template <int TN, bool SWAP, int BK>
__device__ __forceinline__ Unit unit_of(int u, int nt, int tiles, int kb_per, int total_kb) {
  Unit w;
  w.split = u / tiles;
  const int t = u - w.split * tiles;
  const int tm = t / nt, tn = t - tm * nt;
  w.n0 = tn * (SWAP ? 128 : TN);
  w.m0 = tm * (SWAP ? TN : 128);
  w.kb0 = w.split * kb_per;
  w.nkb = min(w.kb0 + kb_per, total_kb) - w.kb0;
  return w;
}

template <int TN, bool SWAP, int BK>
__global__ void __launch_bounds__(THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               int M, int N, int K, int nt, int mt, int splits, int kb_per, int write_hi,
               float alpha, float beta, float *__restrict__ C, int64_t ldc,
               const float *__restrict__ bias, int act, float *__restrict__ ws, int64_t ws_ld,
               int64_t ws_split_stride) {
  using G = typename Pick<TN, SWAP, BK>::G;
  constexpr bool AT = Pick<TN, SWAP, BK>::AT;
  constexpr int S = G::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  constexpr int XB = (AT ? 1 : 2) * G::X_TILE;  // x bytes per stage (AT: no x lo)
  auto x_hi = [&](int s) { return base + s * G::STAGE_BYTES; };
  auto x_lo = [&](int s) { return base + s * G::STAGE_BYTES + G::X_TILE; };
  auto y_hi = [&](int s) { return base + s * G::STAGE_BYTES + XB; };
  auto y_lo = [&](int s) { return base + s * G::STAGE_BYTES + XB + G::Y_TILE; };
  float *staging = reinterpret_cast<float *>(base + S * G::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(base + S * G::STAGE_BYTES + STAGING_BYTES);
  uint64_t *conv = full + S;
  uint64_t *empty = conv + S;
  constexpr int NACC = G::NACC;
  uint64_t *acc_full = empty + S;
  uint64_t *acc_empty = acc_full + NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + NACC);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = nt * mt, units = tiles * splits;
  const int total_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 4);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, G::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the prologue above overlaps the previous kernel's tail (PDL); operands
  // and C are only touched after it has completed
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      // L2 prefetch cursor: walks the same (unit, k-block) sequence as the
      // loads, PF k-blocks ahead, so the ring's TMA loads hit L2 rather than
      // paying HBM latency with only S small stages in flight.
      int pu = blockIdx.x, pkb = 0;
      Unit pw{};
      if (pu < units) pw = unit_of<TN, SWAP, BK>(pu, nt, tiles, kb_per, total_kb);
      auto prefetch_next = [&]() {
        if (pu >= units) return;
        const int kx = (pw.kb0 + pkb) * BK;
        if (!SWAP) {
          ptx::tma_prefetch_2d(&tmA, kx, pw.m0);
          for (int c = 0; c < TN / 32; ++c) ptx::tma_prefetch_2d(&tmB, pw.n0 + 32 * c, kx);
        } else {
          for (int c = 0; c < 4; ++c) ptx::tma_prefetch_2d(&tmB, pw.n0 + 32 * c, kx);
          ptx::tma_prefetch_2d(&tmA, kx, pw.m0);
        }
        if (++pkb == pw.nkb) {
          pkb = 0;
          pu += gridDim.x;
          if (pu < units) pw = unit_of<TN, SWAP, BK>(pu, nt, tiles, kb_per, total_kb);
        }
      };
      const int pf = (write_hi >> 8) & 0xff;
      for (int i = 0; i < pf; ++i) prefetch_next();
      int g = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit w = unit_of<TN, SWAP, BK>(u, nt, tiles, kb_per, total_kb);
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % S;
          if (pf > 0) prefetch_next();
          if (g >= S) ptx::mbar_wait(&empty[s], ((g / S) - 1) & 1);
          if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace) g_trace[0][g] = clock64();
          ptx::mbar_expect_tx(&full[s], G::X_TILE + G::Y_TILE);
          const int kx = (w.kb0 + kb) * BK;
          if (!SWAP) {
            ptx::tma_load_2d(x_hi(s), &tmA, &full[s], kx, w.m0);
#pragma unroll
            for (int c = 0; c < TN / 32; ++c)
              ptx::tma_load_2d(y_hi(s) + c * G::MN_CHUNK, &tmB, &full[s], w.n0 + 32 * c, kx);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              ptx::tma_load_2d(x_hi(s) + c * G::MN_CHUNK, &tmB, &full[s], w.n0 + 32 * c, kx);
            ptx::tma_load_2d(y_hi(s), &tmA, &full[s], kx, w.m0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    {
      // operand A from TMEM has no major-ness (lane = row, column = k)
      constexpr uint32_t idesc = ptx::idesc_tf32(128, TN, SWAP && !AT, !SWAP);
      int g = 0, j = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
        const Unit w = unit_of<TN, SWAP, BK>(u, nt, tiles, kb_per, total_kb);
        const int a = j % NACC;
        if (j >= NACC) ptx::mbar_wait(&acc_empty[a], ((j / NACC) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem + a * TN;
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % S;
          ptx::mbar_wait(&conv[s], (g / S) & 1);
          if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && lane == 0) g_trace[3][g] = clock64();
          ptx::tc_fence_after();
          const uint32_t xh = ptx::smem_u32(x_hi(s)), xl = ptx::smem_u32(x_lo(s));
          const uint32_t yh = ptx::smem_u32(y_hi(s)), yl = ptx::smem_u32(y_lo(s));
          if constexpr (AT) {
            // A hi / lo of this stage in TMEM columns, 8 per k step
            const uint32_t at = tmem + G::A_COL0 + s * 2 * BK;
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              // B: MN-major activations (normal) or K-major weights (swap)
              const uint64_t dyh =
                  SWAP ? ptx::smem_desc(yh + 32 * k, 16, G::K_SBO, G::K_LAYOUT)
                       : ptx::smem_desc(yh + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
              const uint64_t dyl =
                  SWAP ? ptx::smem_desc(yl + 32 * k, 16, G::K_SBO, G::K_LAYOUT)
                       : ptx::smem_desc(yl + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
              if (ACCT_SKIP(write_hi, 4)) continue;
              if (ptx::elect_one()) {
                ptx::mma_tf32_ts(d, at + 8 * k, dyh, idesc, (kb | k) != 0);
                ptx::mma_tf32_ts(d, at + 8 * k, dyl, idesc, 1);
                ptx::mma_tf32_ts(d, at + BK + 8 * k, dyh, idesc, 1);
              }
              __syncwarp();
            }
            if (ptx::elect_one()) ptx::mma_commit(&empty[s]);
            __syncwarp();
            if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && lane == 0) g_trace[4][g] = clock64();
            continue;
          }
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            // K-major: 8 tf32 (32 B) per step inside a row; MN-major
            // SW128_BASE32B: 8 k-rows (two 512-B atoms) per step
            uint64_t dxh, dxl, dyh, dyl;
            if (!SWAP) {
              dxh = ptx::smem_desc(xh + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
              dxl = ptx::smem_desc(xl + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
              dyh = ptx::smem_desc(yh + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
              dyl = ptx::smem_desc(yl + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
            } else {
              dxh = ptx::smem_desc(xh + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
              dxl = ptx::smem_desc(xl + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
              dyh = ptx::smem_desc(yh + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
              dyl = ptx::smem_desc(yl + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
            }
            if (ACCT_SKIP(write_hi, 4)) continue;
            if (ptx::elect_one()) {
              ptx::mma_tf32(d, dxh, dyh, idesc, (kb | k) != 0);
              ptx::mma_tf32(d, dxh, dyl, idesc, 1);
              ptx::mma_tf32(d, dxl, dyh, idesc, 1);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::mma_commit(&empty[s]);
          __syncwarp();
          if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && lane == 0) g_trace[4][g] = clock64();
        }
        if (ptx::elect_one()) ptx::mma_commit(&acc_full[a]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---------------- split hi/lo of each landed stage ----------------
    const int ct = threadIdx.x - 64;  // 0..127
    int g = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit w = unit_of<TN, SWAP, BK>(u, nt, tiles, kb_per, total_kb);
      for (int kb = 0; kb < w.nkb; ++kb, ++g) {
        const int s = g % S;
        ptx::mbar_wait(&full[s], (g / S) & 1);
        if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && ct == 0) g_trace[1][g] = clock64();
        const uint32_t xh = ptx::smem_u32(x_hi(s)), xl = ptx::smem_u32(x_lo(s));
        const uint32_t yh = ptx::smem_u32(y_hi(s)), yl = ptx::smem_u32(y_lo(s));
        if (AT && !(ACCT_SKIP(write_hi, 2))) {
          // operand A (the x tile) -> this stage's TMEM columns, hi then lo.
          // Warp q may write TMEM lanes 32q..32q+31 = MMA rows 32q + lane:
          //  normal: weight row r, its BK values from the SWIZZLE_64B K-major
          //          tile (16-B chunk c of row r at r*64 + (c ^ (r/2 % 4))*16);
          //  swap:   activation column n = 32q + lane of 32-column chunk q,
          //          SWIZZLE_128B_BASE32B MN-major (k-row of 128 B, 32-B
          //          pieces XOR k % 4): one conflict-free 128-B row per k.
          const int q = warp & 3;
          constexpr int NA = BK;  // A values per thread (one MMA row, BK deep)
          uint32_t hi[NA], lo[NA];
          if constexpr (!SWAP) {
            const int row = 32 * q + lane;
            float4 ra[NA / 4];
#pragma unroll
            for (int c = 0; c < NA / 4; ++c)
              ra[c] = ptx::lds128(xh + row * 64 + ((c ^ ((row >> 1) & 3)) << 4));
#pragma unroll
            for (int c = 0; c < NA / 4; ++c) {
              const float v[4] = {ra[c].x, ra[c].y, ra[c].z, ra[c].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t h = __float_as_uint(v[e]) & 0xFFFFE000u;
                hi[4 * c + e] = h;
                lo[4 * c + e] = __float_as_uint(v[e] - __uint_as_float(h));
              }
            }
          } else {
            const uint32_t cb = xh + q * G::MN_CHUNK + ((lane & 7) << 2);
            float va[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k)
              va[k] = ptx::lds32(cb + k * 128 + ((((lane >> 3) ^ k) & 3) << 5));
#pragma unroll
            for (int k = 0; k < NA; ++k) {
              const uint32_t h = __float_as_uint(va[k]) & 0xFFFFE000u;
              hi[k] = h;
              lo[k] = __float_as_uint(va[k] - __uint_as_float(h));
            }
          }
          constexpr int NY = (G::Y_TILE / 16 + 127) / 128;
          float4 ry[NY];
#pragma unroll
          for (int i = 0; i < NY; ++i)
            if (ct + 128 * i < G::Y_TILE / 16) ry[i] = ptx::lds128(yh + 16 * (ct + 128 * i));
          const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + G::A_COL0 + s * 2 * BK;
          ptx::tmem_st_cols<NA>(ta, hi);
          ptx::tmem_st_cols<NA>(ta + BK, lo);
#pragma unroll
          for (int i = 0; i < NY; ++i) {
            if (ct + 128 * i < G::Y_TILE / 16) {
              float4 h4;
              ptx::sts128(yl + 16 * (ct + 128 * i), split_lo(ry[i], h4));
            }
          }
          ptx::tmem_st_wait();
        } else if (!(ACCT_SKIP(write_hi, 2))) {
          // every load of the stage in flight before the first store
          constexpr int NX = G::X_TILE / 16 / 128;
          constexpr int NY = (G::Y_TILE / 16 + 127) / 128;
          float4 rx[NX], ry[NY];
#pragma unroll
          for (int i = 0; i < NX; ++i) rx[i] = ptx::lds128(xh + 16 * (ct + 128 * i));
#pragma unroll
          for (int i = 0; i < NY; ++i)
            if (ct + 128 * i < G::Y_TILE / 16) ry[i] = ptx::lds128(yh + 16 * (ct + 128 * i));
          if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && ct == 0)
            g_trace[5][g] = clock64() + (long long)(rx[0].x * 0.0f) + (long long)(ry[0].x * 0.0f);
#pragma unroll
          for (int i = 0; i < NX; ++i) {
            float4 hi;
            ptx::sts128(xl + 16 * (ct + 128 * i), split_lo(rx[i], hi));
            if (write_hi & 1) ptx::sts128(xh + 16 * (ct + 128 * i), hi);
          }
#pragma unroll
          for (int i = 0; i < NY; ++i) {
            if (ct + 128 * i < G::Y_TILE / 16) {
              float4 hi;
              ptx::sts128(yl + 16 * (ct + 128 * i), split_lo(ry[i], hi));
              if (write_hi & 1) ptx::sts128(yh + 16 * (ct + 128 * i), hi);
            }
          }
        }
        if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && ct == 0) g_trace[6][g] = clock64();
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> tensor core
        if (AT) ptx::tc_fence_before();  // tcgen05.st -> the MMA issuer's thread sync
        if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && ct == 0) g_trace[7][g] = clock64();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&conv[s]);
        if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace && ct == 0) g_trace[2][g] = clock64();
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // this warp may read TMEM lanes 32q..32q+31
    const int grp = (warp - 6) / 4;
    const uint32_t stg_s = ptx::smem_u32(staging + (grp * 4 + q) * (32 * 33));
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      if ((j % EPI_GROUPS) != grp) continue;
      const Unit w = unit_of<TN, SWAP, BK>(u, nt, tiles, kb_per, total_kb);
      const int a = j % NACC;
      ptx::mbar_wait(&acc_full[a], (j / NACC) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + a * TN;
      float *part = ws + w.split * ws_split_stride;
      if (ACCT_SKIP(write_hi, 8)) {
        // debug: skip the epilogue body
      } else if (!SWAP) {
        // lanes = output rows: transpose each 32x32 chunk through smem so that
        // lane = column and each store writes a contiguous 128-B row segment
        const int row0 = w.m0 + 32 * q;
        for (int c = 0; c < TN / 32; ++c) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(trow + 32 * c, r);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) ptx::sts32(stg_s + 4 * (lane * 33 + jj), __uint_as_float(r[jj]));
          __syncwarp();
          const int col = w.n0 + 32 * c + lane;
          if (splits == 1) {
            // bias of row row0+i is loaded once by lane i, then broadcast
            const float my_bias = (bias && row0 + lane < M) ? __ldg(bias + row0 + lane) : 0.0f;
            float bv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) bv[i] = __shfl_sync(0xffffffffu, my_bias, i);
            if (col < N) {
              float cv[32];
#pragma unroll
              for (int i = 0; i < 32; ++i)  // all C loads in flight before any store
                cv[i] = (beta != 0.0f && row0 + i < M) ? C[(int64_t)(row0 + i) * ldc + col] : 0.0f;
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                v[i] = finish_lin(ptx::lds32(stg_s + 4 * (i * 33 + lane)), alpha, beta, cv[i], bias,
                                  bv[i]);
              if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (row0 + i < M) C[(int64_t)(row0 + i) * ldc + col] = v[i];
            }
          } else {
            float *dst = part + (int64_t)row0 * ws_ld + col;
#pragma unroll 8
            for (int i = 0; i < 32; ++i)
              __stcg(dst + (int64_t)i * ws_ld, ptx::lds32(stg_s + 4 * (i * 33 + lane)));
          }
          __syncwarp();
        }
      } else {
        // lanes = output columns, TMEM columns = output rows
        const int col = w.n0 + 32 * q + lane;
        constexpr int CH = 16;  // 16 rows per TMEM load keeps the epilogue in registers
        for (int c = 0; c < TN / CH; ++c) {
          uint32_t r[CH];
          ptx::tmem_ld_32x32b_x16(trow + CH * c, r);
          if (col >= N) continue;
          const int rbase = w.m0 + CH * c;
          if (splits == 1) {
            float cv[CH], bv[CH];
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) {  // every load in flight before any store
              const bool ok = rbase + jj < M;
              cv[jj] = (beta != 0.0f && ok) ? C[(int64_t)(rbase + jj) * ldc + col] : 0.0f;
              bv[jj] = (bias && ok) ? __ldg(bias + rbase + jj) : 0.0f;
            }
            float v[CH];
#pragma unroll
            for (int jj = 0; jj < CH; ++jj)
              v[jj] = finish_lin(__uint_as_float(r[jj]), alpha, beta, cv[jj], bias, bv[jj]);
            if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
            for (int jj = 0; jj < CH; ++jj)
              if (rbase + jj < M) C[(int64_t)(rbase + jj) * ldc + col] = v[jj];
          } else {
            float *dst = part + (int64_t)rbase * ws_ld + col;
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) __stcg(dst + (int64_t)jj * ws_ld, __uint_as_float(r[jj]));
          }
        }
      }
      // accumulator a may be overwritten once all four warps have read it
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[a]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, G::TMEM_COLS);
}

// ------------------------------------------------------------------ CTA pairs
// 2-CTA (cta_group::2) variant of the normal orientation: a CTA pair computes
// a 256 x TN tile -- CTA r owns weight rows m0 + 128 r (operand A, hi/lo in
// its own TMEM) and B columns n0 + r TN/2 .. (its half of operand B, raw + lo
// in its shared memory).  The leader (rank 0) issues
// `tcgen05.mma.cta_group::2` with M = 256; each tensor core reads its own B
// half and the pair exchanges them, so per SM and 16-deep k-block the
// shared-memory traffic is TMA 8 + TN/8 KB, split 8 + TN/8...:
// 52 KB at TN = 192 against 576 MMA cycles, under the 128 B/clk port.
// Synchronisation:
//   full[s]      local: TMA bytes of this CTA's stage landed
//   conv[s]      LEADER: split done in both CTAs (8 warp arrivals, cluster scope)
//   empty[s]     local in both: MMA commit multicast to the pair
//   acc_full[a]  local in both: unit's last MMA commit multicast
//   acc_empty[a] LEADER: both CTAs' epilogue warps drained accumulator a (8)
__device__ __forceinline__ long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}

// SWAP (M <= 64 weight rows): operand A = 128 activation COLUMNS per CTA
// (256 per pair, transposed into TMEM by the split warps), operand B = the
// TN weight rows, TN/2 per CTA, K-major; the epilogue writes lanes = columns.
// DUAL: the two small 3xTF32 terms (hi.lo + lo.hi) accumulate in their own
// TMEM accumulator next to hi.hi and the epilogue adds the two in FP32.  The
// tensor core's FP32 accumulate truncates; folding the small terms into the
// big accumulator costs three truncations of it per k step instead of one.
// LOA: only A lo goes to TMEM (BK columns per stage instead of 2 BK); the MMAs
// with A hi read the raw K-major tile from shared memory -- leaves TMEM room
// for DUAL with BK = 32
// IMB (implicit B, with PK): operand B is the im2col of a 3x3 / stride 1 /
// pad 1 convolution's input, gathered by the split warps straight from the
// input planes (L2-resident: 11 MB for yolov2-tiny L13 at 16 images) instead
// of a col array that an im2col launch wrote to HBM and TMA reads back.  B
// column n of the launch = image n / img, pixel n % img (the interleaved
// multi-image layout); row k = (channel k / 9, tap k % 9).  The gathered
// values are the col array's exactly, so C is bit-identical to im2col + the
// same gemm, and the split warps store them to col for the images whose col
// is observable (n >= col_n0).
struct ImB {
  const float *act;         // conv input: channel c of image b at act + c act_ld + b act_img
  int64_t act_ld, act_img;
  int64_t img;              // launch column pitch of one image (0: one image)
  int cin, H, W;            // input planes (= output planes: 3x3 / 1 / 1)
  float *col;               // col array (null: no column observable)
  int64_t col_ld, col_n0;   // col row stride; first launch column whose col is stored
};

// PK > 0 (chunked promotion): the k-loop of a unit is cut into chunks of PK
// k-blocks; each chunk accumulates into a FRESH TMEM accumulator (two,
// ping-pong, NACC = 2) and BOTH epilogue groups add the finished chunk into
// an FP32 running sum in registers (group g: columns g TN/2 .. of its 128
// rows), rounding to nearest.  The tensor core's truncating accumulate then
// compounds over PK k-blocks instead of the whole K (K = 9216: 48 vs 1152
// truncations of the big accumulator) -- the long-K layers' error falls
// ~20x below DUAL's.  The unit's final store overlaps the next unit's first
// chunk (the other accumulator).
template <int TN, int NACC_, int BK_, bool SWAP_ = false, bool DUAL_ = false, bool LOA_ = false,
          int PK_ = 0, bool IMB_ = false>
struct Cfg2 {
  static constexpr int PK = PK_;
  // implicit B: per stage, the input slab the k-block's B rows are gathered
  // from -- SLAB_CH channels x SEG consecutive pixels, for up to two images
  static constexpr int SEG = 256, SLAB_CH = 5;
#ifdef ACCT_DBG_NOSLAB
  static constexpr int SLAB_BYTES = 0;
#else
  static constexpr int SLAB_BYTES = IMB_ ? 2 * SLAB_CH * SEG * 4 : 0;
#endif
  static_assert(PK_ == 0 || (!SWAP_ && !DUAL_ && NACC_ == 2 && TN == 192),
                "chunked promotion: normal 192-wide pair tile, two accumulators");
  static constexpr bool SWAP = SWAP_;
  static constexpr bool DUAL = DUAL_;
  static constexpr bool LOA = LOA_;
  static constexpr int A_STAGE_COLS = (LOA_ ? 1 : 2) * BK_;
  static constexpr int ACC = (DUAL_ ? 2 : 1) * TN;   // TMEM columns per accumulator slot
  static constexpr int BK = BK_;
  static constexpr int HALF = TN / 2;
  static constexpr int X_TILE = 128 * BK * 4;
  static constexpr int Y_TILE = HALF * BK * 4;
  static constexpr uint32_t K_SBO = 8 * BK * 4;  // 8-row swizzle atom of a K-major tile
  static constexpr uint32_t K_LAYOUT = BK == 32 ? ptx::kLayoutSW128 : 4u;
  static constexpr int STAGE_BYTES = X_TILE + 2 * Y_TILE + SLAB_BYTES;
  static constexpr int NACC = NACC_;
  static constexpr int BUDGET = 220 * 1024 - STAGING_BYTES - 512 - 1024;
  static constexpr int SMEM_STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  static constexpr int TMEM_STAGES = (512 - NACC * ACC) / A_STAGE_COLS;
#ifdef ACCT_DBG_S3
  static constexpr int STAGES = 3;
#else
  static constexpr int STAGES = SMEM_STAGES < TMEM_STAGES ? SMEM_STAGES : TMEM_STAGES;
#endif
  static constexpr int A_COL0 = NACC * ACC;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 512 + 1024;
  static constexpr uint32_t MN_CHUNK = BK * 128;
  static constexpr int ROWB = BK * 4;  // K-major A row bytes: 64 (SWIZZLE_64B) or 128 (128B)
  static_assert(BK == 16 || BK == 32, "BK");
  static_assert(SWAP ? HALF % 8 == 0 : HALF % 32 == 0, "operand B half tile shape");
  static_assert(STAGES >= 2, "pipeline too shallow");
};

template <int TN, int NACC, int BK_, bool SWAP, bool DUAL = false, bool LOA = false, int PK = 0,
          bool IMB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
tc2_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int M, int N, int K, int nt, int mt, int splits, int kb_per, int write_hi,
                float alpha, float beta, float *__restrict__ C, int64_t ldc,
                const float *__restrict__ bias, int act, float *__restrict__ ws, int64_t ws_ld,
                int64_t ws_split_stride, int *__restrict__ sk_flags, const ImB imb) {
  using G = Cfg2<TN, NACC, BK_, SWAP, DUAL, LOA, PK, IMB>;
  static_assert(!IMB || (PK > 0 && !SWAP), "implicit B: the chunked-promotion normal tile");
  constexpr int S = G::STAGES, BK = G::BK;
  static_assert(!LOA || !SWAP, "LOA is for the normal orientation");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  auto x_hi = [&](int s) { return base + s * G::STAGE_BYTES; };
  auto y_hi = [&](int s) { return base + s * G::STAGE_BYTES + G::X_TILE; };
  auto y_lo = [&](int s) { return base + s * G::STAGE_BYTES + G::X_TILE + G::Y_TILE; };
  auto slab = [&](int s) { return base + s * G::STAGE_BYTES + G::X_TILE + 2 * G::Y_TILE; };

  float *staging = reinterpret_cast<float *>(base + S * G::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(base + S * G::STAGE_BYTES + STAGING_BYTES);
  uint64_t *conv = full + S;
  uint64_t *empty = conv + S;
  uint64_t *acc_full = empty + S;
  uint64_t *acc_empty = acc_full + NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + NACC);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_rank();
  const int pair = blockIdx.x / 2, pairs = gridDim.x / 2;
  const int tiles = nt * mt, units = tiles * splits;
  const int total_kb = (K + BK - 1) / BK;
  auto unit = [&](int u) {
    Unit w;
    w.split = u / tiles;
    const int t = u - w.split * tiles;
    const int tm = t / nt, tn = t - tm * nt;
    w.n0 = tn * (SWAP ? 256 : TN);
    w.m0 = tm * (SWAP ? TN : 256);
    w.kb0 = w.split * kb_per;
    w.nkb = min(w.kb0 + kb_per, total_kb) - w.kb0;
    return w;
  };
  // Stream-K (PK > 0): the space of (tile, chunk of PK k-blocks) is cut into
  // `pairs` equal contiguous ranges, one per CTA pair, so every pair does the
  // same MMA work whatever tiles / pairs is (yolov2-608 L23: 124 tiles on 74
  // pairs).  A pair's range is a list of segments (tile, chunks [c0, c1)); a
  // tile cut between pairs is completed by whichever of its segments counts
  // in last (workspace slots + a per-tile counter, see the epilogue).
  const int cpt = PK > 0 ? (total_kb + PK - 1) / PK : 1;
  const int64_t tot_ch = (int64_t)tiles * cpt;
  const int64_t sk_begin = tot_ch * pair / pairs, sk_end = tot_ch * (pair + 1) / pairs;
  auto seg_at = [&](int64_t pos, Unit &w, int &c0, int &c1) {
    const int t = (int)(pos / cpt);
    c0 = (int)(pos - (int64_t)t * cpt);
    const int64_t rem = sk_end - pos;
    c1 = rem < (int64_t)(cpt - c0) ? c0 + (int)rem : cpt;
    const int tm = t / nt, tn = t - tm * nt;
    w.split = t;  // the tile index
    w.n0 = tn * TN;
    w.m0 = tm * 256;
    w.kb0 = c0 * (PK > 0 ? PK : 1);
    w.nkb = min(c1 * (PK > 0 ? PK : 1), total_kb) - w.kb0;
  };
  // every role walks the same work list: stream-K segments or split units
  const bool sk = PK > 0 && sk_flags != nullptr;  // else split units (maybe split-K)
  auto for_each_unit = [&](auto &&body) {
    if (!sk) {
      for (int u = pair; u < units; u += pairs) {
        const Unit w = unit(u);
        body(w, 0, (w.nkb + (PK > 0 ? PK : 1) - 1) / (PK > 0 ? PK : 1));
      }
    } else {
      for (int64_t pos = sk_begin; pos < sk_end;) {
        Unit w;
        int c0, c1;
        seg_at(pos, w, c0, c1);
        body(w, c0, c1);
        pos += c1 - c0;
      }
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 8);  // leader: 4 split warps of each CTA
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], PK ? 16 : 8);  // epilogue warps of both CTAs
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc2(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  // implicit B: the images a unit's half tile (this CTA's HALF columns)
  // touches -- at most two (the host requires an image pitch >= HALF) -- and
  // the 16-B aligned first pixel of each image's slab segment
  struct Span {
    int b0, nimg, start[2];
  };
  auto span_of = [&](const Unit &w) {
    Span sp{0, 0, {0, 0}};
    const int n_first = w.n0 + rank * G::HALF;
    const int n_last = min(n_first + G::HALF, N) - 1;
    if (n_first > n_last) return sp;
    const int img = (int)imb.img;
    sp.b0 = img ? n_first / img : 0;
    const int b1 = img ? n_last / img : 0;
    sp.nimg = b1 - sp.b0 + 1;
    for (int t = 0; t < sp.nimg; ++t) {
      const int p_lo = t == 0 ? n_first - sp.b0 * img : 0;
      sp.start[t] = max(0, p_lo - imb.W - 1) & ~3;
    }
    return sp;
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: their own A rows, B half) ----------------
    if (lane == 0) {
      int g = 0;
      for_each_unit([&](const Unit &w, int, int) {
        const int m_rows = w.m0 + (SWAP ? rank * G::HALF : 128 * rank);
        const int n_cols = w.n0 + (SWAP ? 128 * rank : rank * G::HALF);
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % S;
          if (g >= S) ptx::mbar_wait(&empty[s], ((g / S) - 1) & 1);
          if ((write_hi & 16) && blockIdx.x == 0 && g < kTrace) g_trace[0][g] = gtimer();
          const int kx = (w.kb0 + kb) * BK;
          if constexpr (IMB) {
            // A, and the input slab segments of the k-block's <= 5 channels
            // (tmB = the input as (pixels, images, channels), zeros past the
            // plane and past the channels)
            const Span sp = span_of(w);
            const int nload = ACCT_SKIP(write_hi, 32) ? 0 : sp.nimg;  // profiling: no slab TMA
            ptx::mbar_expect_tx(&full[s], G::X_TILE + nload * G::SLAB_CH * G::SEG * 4);
            ptx::tma_load_2d(x_hi(s), &tmA, &full[s], kx, m_rows);
            for (int t = 0; t < nload; ++t)
              ptx::tma_load_3d(slab(s) + t * G::SLAB_CH * G::SEG * 4, &tmB, &full[s], sp.start[t],
                               sp.b0 + t, kx / 9);
          } else if constexpr (!SWAP) {
            ptx::mbar_expect_tx(&full[s], G::X_TILE + G::Y_TILE);
            ptx::tma_load_2d(x_hi(s), &tmA, &full[s], kx, m_rows);
#pragma unroll
            for (int c = 0; c < G::HALF / 32; ++c)
              ptx::tma_load_2d(y_hi(s) + c * G::MN_CHUNK, &tmB, &full[s], n_cols + 32 * c, kx);
          } else {
            ptx::mbar_expect_tx(&full[s], G::X_TILE + G::Y_TILE);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              ptx::tma_load_2d(x_hi(s) + c * G::MN_CHUNK, &tmB, &full[s], n_cols + 32 * c, kx);
            ptx::tma_load_2d(y_hi(s), &tmA, &full[s], kx, m_rows);
          }
        }
      });
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only; whole warp, one lane issues) ----------------
    if (rank == 0 && PK > 0) {
      // chunked promotion: chunk c (counted across units) -> accumulator c & 1
      constexpr uint32_t idesc = ptx::idesc_tf32(256, TN, false, true);
      int g = 0, c = 0;
      for_each_unit([&](const Unit &w, int, int) {
        uint32_t d = tmem;
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int kc = kb % (PK > 0 ? PK : 1);
          if (kc == 0) {
            if (c >= 2) ptx::mbar_wait_cluster(&acc_empty[c & 1], ((c >> 1) - 1) & 1);
            ptx::tc_fence_after();
            d = tmem + (c & 1) * G::ACC;
          }
          const int s = g % S;
          ptx::mbar_wait(&conv[s], (g / S) & 1);
          ptx::tc_fence_after();
          const uint32_t yh = ptx::smem_u32(y_hi(s)), yl = ptx::smem_u32(y_lo(s));
          const uint32_t at = tmem + G::A_COL0 + s * G::A_STAGE_COLS;
          const uint32_t xhs = ptx::smem_u32(x_hi(s));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t dyh = ptx::smem_desc(yh + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
            const uint64_t dyl = ptx::smem_desc(yl + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
            if (ACCT_SKIP(write_hi, 4)) continue;
            if (ptx::elect_one()) {
              if constexpr (LOA) {
                const uint64_t dxh = ptx::smem_desc(xhs + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
                ptx::mma2_tf32_ss(d, dxh, dyh, idesc, (kc | k) != 0);
                ptx::mma2_tf32_ss(d, dxh, dyl, idesc, 1);
                ptx::mma2_tf32_ts(d, at + 8 * k, dyh, idesc, 1);
              } else {
                ptx::mma2_tf32_ts(d, at + 8 * k, dyh, idesc, (kc | k) != 0);
                ptx::mma2_tf32_ts(d, at + 8 * k, dyl, idesc, 1);
                ptx::mma2_tf32_ts(d, at + BK + 8 * k, dyh, idesc, 1);
              }
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::mma2_commit_multicast(&empty[s], 0x3);
          __syncwarp();
          if (kc == PK - 1 || kb == w.nkb - 1) {
            if (ptx::elect_one()) ptx::mma2_commit_multicast(&acc_full[c & 1], 0x3);
            __syncwarp();
            ++c;
          }
        }
      });
    } else if (rank == 0) {
      constexpr uint32_t idesc = ptx::idesc_tf32(256, TN, false, !SWAP);
      int g = 0, j = 0;
      for (int u = pair; u < units; u += pairs, ++j) {
        const Unit w = unit(u);
        const int a = j % NACC;
        if (j >= NACC) ptx::mbar_wait_cluster(&acc_empty[a], ((j / NACC) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem + a * G::ACC;
        const uint32_t d2 = DUAL ? d + TN : d;  // small-term accumulator
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % S;
          ptx::mbar_wait(&conv[s], (g / S) & 1);
          if ((write_hi & 16) && g < kTrace && blockIdx.x == 0 && lane == 0)
            g_trace[3][g] = gtimer();
          ptx::tc_fence_after();
          const uint32_t yh = ptx::smem_u32(y_hi(s)), yl = ptx::smem_u32(y_lo(s));
          const uint32_t at = tmem + G::A_COL0 + s * G::A_STAGE_COLS;
          const uint32_t xhs = ptx::smem_u32(x_hi(s));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t dyh =
                SWAP ? ptx::smem_desc(yh + 32 * k, 16, G::K_SBO, G::K_LAYOUT)
                     : ptx::smem_desc(yh + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
            const uint64_t dyl =
                SWAP ? ptx::smem_desc(yl + 32 * k, 16, G::K_SBO, G::K_LAYOUT)
                     : ptx::smem_desc(yl + 1024 * k, G::MN_CHUNK, 512, ptx::kLayoutSW128Base32B);
            if (ACCT_SKIP(write_hi, 4)) continue;
            if (ptx::elect_one()) {
              if constexpr (LOA) {
                // A hi = the raw K-major tile in shared memory, A lo in TMEM
                const uint64_t dxh = ptx::smem_desc(xhs + 32 * k, 16, G::K_SBO, G::K_LAYOUT);
                ptx::mma2_tf32_ss(d, dxh, dyh, idesc, (kb | k) != 0);
                ptx::mma2_tf32_ss(d2, dxh, dyl, idesc, DUAL ? (kb | k) != 0 : 1);
                ptx::mma2_tf32_ts(d2, at + 8 * k, dyh, idesc, 1);
              } else {
                ptx::mma2_tf32_ts(d, at + 8 * k, dyh, idesc, (kb | k) != 0);
                ptx::mma2_tf32_ts(d2, at + 8 * k, dyl, idesc, DUAL ? (kb | k) != 0 : 1);
                ptx::mma2_tf32_ts(d2, at + BK + 8 * k, dyh, idesc, 1);
              }
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::mma2_commit_multicast(&empty[s], 0x3);
          __syncwarp();
          if ((write_hi & 16) && g < kTrace && blockIdx.x == 0 && lane == 0)
            g_trace[4][g] = gtimer();
        }
        if (ptx::elect_one()) ptx::mma2_commit_multicast(&acc_full[a], 0x3);
        __syncwarp();
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---------------- split (both CTAs): A -> own TMEM hi/lo, B half lo ----------------
    const int ct = threadIdx.x - 64;
    const int q = warp & 3, row = 32 * q + lane;
    const uint32_t conv_leader = ptx::mapa(ptx::smem_u32(&conv[0]), 0);
    int g = 0;
    for_each_unit([&](const Unit &w, int, int) {
      // implicit B: this thread gathers columns 3 lane .. 3 lane + 2 of the
      // CTA's half tile, rows q, q + 4, ... of every k-block
      // (column 32 j + lane of the half tile = launch column n = image
      // n / img, pixel n % img: its slab offset, the 9-bit mask of its taps
      // inside the plane, whether its col is stored)
      int goff[3], gn[3];
      uint32_t gmask[3];
      bool gcol[3];
      if constexpr (IMB) {
        const int HW = imb.H * imb.W;
        const Span sp = span_of(w);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int n = w.n0 + rank * G::HALF + 32 * j + lane;
          const int im = imb.img ? (int)(n / imb.img) : 0;
          const int px = n - (int)(im * imb.img);
          const int t = im - sp.b0;
          const bool ok = n < N && px < HW && t >= 0 && t < sp.nimg;
          const int y = px / imb.W, x = px - (px / imb.W) * imb.W;
          uint32_t m = 0;
#pragma unroll
          for (int r = 0; r < 9; ++r) {
            const int yy = y + r / 3 - 1, xx = x + r % 3 - 1;
            if (ok && yy >= 0 && yy < imb.H && xx >= 0 && xx < imb.W) m |= 1u << r;
          }
          gmask[j] = m;
          gn[j] = n;
          gcol[j] = ok && imb.col != nullptr && n >= imb.col_n0;
          goff[j] = t * G::SLAB_CH * G::SEG + px - sp.start[t & 1];
        }
      }
      for (int kb = 0; kb < w.nkb; ++kb, ++g) {
        const int s = g % S;
        ptx::mbar_wait(&full[s], (g / S) & 1);
        if ((write_hi & 16) && blockIdx.x < 2 && g < kTrace && ct == 0)
          g_trace[blockIdx.x == 0 ? 1 : 5][g] = gtimer();
        const uint32_t xh = ptx::smem_u32(x_hi(s));
        const uint32_t yh = ptx::smem_u32(y_hi(s)), yl = ptx::smem_u32(y_lo(s));
        if constexpr (IMB) {
          // B from the slab: raw and lo of each value at its
          // SWIZZLE_128B_BASE32B place (32-column chunks, 128-B rows, 32-B
          // pieces XOR k % 4); col for the observable images
          const int kx = (w.kb0 + kb) * BK;
          const int K9 = 9 * imb.cin;
          const int c0 = kx / 9;
          const uint32_t sl = ptx::smem_u32(slab(s));
          // lane = one column of each 32-column chunk: conflict-free LDS
          // (consecutive pixels) and STS (one 128-B row per chunk and k)
          const uint32_t lane_off = (uint32_t)((lane & 7) << 2);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int kl = q + 4 * i;
            const int k = kx + kl;
            const int c = k / 9, r = k - 9 * c;
            const int tap = (c - c0) * G::SEG + (r / 3 - 1) * imb.W + (r - 3 * (r / 3)) - 1;
            const uint32_t row = kl * 128 + ((((lane >> 3) ^ kl) & 3) << 5) + lane_off;
            const bool kin = k < K9;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const bool ok = kin && ((gmask[j] >> r) & 1u);
              const float v = ok && !ACCT_SKIP(write_hi, 64) ? ptx::lds32(sl + 4 * (goff[j] + tap))
                                                             : 0.0f;
              const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
              ptx::sts32(yh + j * G::MN_CHUNK + row, v);
              ptx::sts32(yl + j * G::MN_CHUNK + row, v - h);
              if (gcol[j] && kin) __stcs(imb.col + (int64_t)k * imb.col_ld + gn[j], v);
            }
          }
        }
        if (!(ACCT_SKIP(write_hi, 2))) {
          // row r of the K-major A tile: 16-B chunk c at r*ROWB + (c ^ swz(r))*16,
          // swz = (r/2)%4 for SWIZZLE_64B rows, r%8 for SWIZZLE_128B rows
          // swap: activation column 32q + lane of chunk q, one conflict-free
          // 128-B SWIZZLE_128B_BASE32B row per k (32-B pieces XOR k % 4)
          float4 ra[BK / 4];
          if constexpr (!SWAP) {
#pragma unroll
            for (int c = 0; c < BK / 4; ++c)
              ra[c] = ptx::lds128(xh + row * G::ROWB +
                                  ((c ^ (BK == 16 ? ((row >> 1) & 3) : (row & 7))) << 4));
          } else {
            const uint32_t cb = xh + q * G::MN_CHUNK + ((lane & 7) << 2);
#pragma unroll
            for (int c = 0; c < BK / 4; ++c) {
              float v[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int kk = 4 * c + e;
                v[e] = ptx::lds32(cb + kk * 128 + ((((lane >> 3) ^ kk) & 3) << 5));
              }
              ra[c] = make_float4(v[0], v[1], v[2], v[3]);
            }
          }
          constexpr int NY = IMB ? 1 : (G::Y_TILE / 16 + 127) / 128;
          float4 ry[NY];
          if constexpr (!IMB) {
#pragma unroll
            for (int i = 0; i < NY; ++i)
              if (ct + 128 * i < G::Y_TILE / 16) ry[i] = ptx::lds128(yh + 16 * (ct + 128 * i));
          }
          uint32_t hi[BK], lo[BK];
#pragma unroll
          for (int c = 0; c < BK / 4; ++c) {
            const float v[4] = {ra[c].x, ra[c].y, ra[c].z, ra[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t h = __float_as_uint(v[e]) & 0xFFFFE000u;
              hi[4 * c + e] = h;
              lo[4 * c + e] = __float_as_uint(v[e] - __uint_as_float(h));
            }
          }
          const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + G::A_COL0 + s * G::A_STAGE_COLS;
          if constexpr (LOA) {
            ptx::tmem_st_cols<BK>(ta, lo);
          } else {
            ptx::tmem_st_cols<BK>(ta, hi);
            ptx::tmem_st_cols<BK>(ta + BK, lo);
          }
          if constexpr (!IMB) {
#pragma unroll
            for (int i = 0; i < NY; ++i) {
              if (ct + 128 * i < G::Y_TILE / 16) {
                float4 h4;
                ptx::sts128(yl + 16 * (ct + 128 * i), split_lo(ry[i], h4));
              }
            }
          }
          ptx::tmem_st_wait();
        }
        ptx::fence_proxy_async_smem();  // B lo -> the pair's tensor cores
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(conv_leader + 8 * s);
        if ((write_hi & 16) && blockIdx.x < 2 && g < kTrace && ct == 0)
          g_trace[blockIdx.x == 0 ? 2 : 6][g] = gtimer();
      }
    });
  } else if constexpr (PK > 0) {
    // ---------------- epilogue, chunked promotion (both CTAs, both groups) ----------------
    // group grp owns columns grp HC .. of the CTA's 128 rows: every chunk is
    // added into an FP32 running sum in registers, then the sum goes out
    // through the warp's staging transpose like the plain epilogue
    constexpr int HC = TN / 2;
    const int q = warp & 3;
    const int grp = (warp - 6) / 4;
    const uint32_t stg_s = ptx::smem_u32(staging + (grp * 4 + q) * (32 * 33));
    const uint32_t acc_empty_leader = ptx::mapa(ptx::smem_u32(&acc_empty[0]), 0);
    int c = 0;
    const int row = 32 * q + lane;  // this thread's row of the CTA's 128
    for_each_unit([&](const Unit &w, int c0, int c1) {
      const int nch = c1 - c0;
      float acc[HC];
#pragma unroll
      for (int i = 0; i < HC; ++i) acc[i] = 0.0f;
      for (int ci = 0; ci < nch; ++ci, ++c) {
        const int a = c & 1;
        ptx::mbar_wait(&acc_full[a], (c >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + a * G::ACC + grp * HC;
#pragma unroll
        for (int p = 0; p < HC / 16; ++p) {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(trow + 16 * p, r);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) acc[16 * p + jj] += __uint_as_float(r[jj]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(acc_empty_leader + 8 * a);
      }
      if (ACCT_SKIP(write_hi, 8)) return;
      constexpr int SLOT = 128 * TN;  // one CTA's partial tile in the workspace
      if (sk && (c0 > 0 || c1 < cpt)) {
        // a tile cut between pairs: every segment leaves its partial sum in
        // its slot (two per CTA: the tile its range starts in, the tile it
        // ends in), then counts itself in with one acq_rel atomic per CTA;
        // the segment that completes the count sums the tile's partials in
        // pair order (deterministic whoever arrives last) and finishes it.
        // Nothing ever waits for another CTA, so any number of launches may
        // share the GPU.
        const int t = w.split;
        const int64_t tile_lo = (int64_t)t * cpt, tile_hi = tile_lo + cpt;
        auto pair_of = [&](int64_t chunk) {  // the pair whose range holds chunk
          int qp = (int)(chunk * pairs / tot_ch);
          while (qp + 1 < pairs && tot_ch * (qp + 1) / pairs <= chunk) ++qp;
          while (qp > 0 && tot_ch * qp / pairs > chunk) --qp;
          return qp;
        };
        auto slot_of = [&](int qp) {  // 0: the tile the pair's range starts in
          const int first_tile = (int)((tot_ch * qp / pairs) / cpt);
          return 2 * (2 * qp + (int)rank) + (t == first_tile ? 0 : 1);
        };
        const int q_first = pair_of(tile_lo), q_last = pair_of(tile_hi - 1);
        float *mine = ws + (int64_t)slot_of(pair) * SLOT + (int64_t)row * TN + grp * HC;
#pragma unroll
        for (int i = 0; i < HC / 4; ++i)
          __stcg(reinterpret_cast<float4 *>(mine) + i,
                 make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]));
        __threadfence();
        asm volatile("bar.sync 3, 256;" ::: "memory");  // the eight epilogue warps
        volatile uint32_t *last_flag = tmem_slot + 1;
        if (threadIdx.x == 6 * 32) {
          int old;
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                       : "=r"(old) : "l"(sk_flags + 2 * t + rank) : "memory");
          const bool last = old == q_last - q_first;
          if (last) sk_flags[2 * t + rank] = 0;  // zero for the next launch on this stream
          *last_flag = last ? 1u : 0u;
        }
        asm volatile("bar.sync 3, 256;" ::: "memory");
        if (*last_flag == 0u) return;
        __threadfence();
#pragma unroll
        for (int i = 0; i < HC; ++i) acc[i] = 0.0f;
        for (int qp = q_first; qp <= q_last; ++qp) {
          const float *slot = ws + (int64_t)slot_of(qp) * SLOT + (int64_t)row * TN + grp * HC;
#pragma unroll
          for (int i = 0; i < HC / 4; ++i) {
            const float4 v = __ldcg(reinterpret_cast<const float4 *>(slot) + i);
            acc[4 * i] += v.x;
            acc[4 * i + 1] += v.y;
            acc[4 * i + 2] += v.z;
            acc[4 * i + 3] += v.w;
          }
        }
      }
      const int row0 = w.m0 + 128 * rank + 32 * q;
#pragma unroll
      for (int cb = 0; cb < HC / 32; ++cb) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) ptx::sts32(stg_s + 4 * (lane * 33 + jj), acc[32 * cb + jj]);
        __syncwarp();
        const int col = w.n0 + grp * HC + 32 * cb + lane;
        if (!sk && splits > 1) {
          float *dst = ws + w.split * ws_split_stride + (int64_t)row0 * ws_ld + col;
#pragma unroll 8
          for (int i = 0; i < 32; ++i)
            __stcg(dst + (int64_t)i * ws_ld, ptx::lds32(stg_s + 4 * (i * 33 + lane)));
        } else {
          if (col < N) {
            // 8 rows at a time: the 96-float running sum stays in registers
#pragma unroll 1
            for (int i0 = 0; i0 < 32; i0 += 8) {
              float v[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int orow = row0 + i0 + i;
                const bool ok = orow < M;
                // one broadcast load per row (every lane reads the same bias)
                const float bv = bias && ok ? __ldg(bias + orow) : 0.0f;
                const float cv = beta != 0.0f && ok ? C[(int64_t)orow * ldc + col] : 0.0f;
                v[i] = finish_lin(ptx::lds32(stg_s + 4 * ((i0 + i) * 33 + lane)), alpha, beta, cv,
                                  bias, bv);
              }
              if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (row0 + i0 + i < M) C[(int64_t)(row0 + i0 + i) * ldc + col] = v[i];
            }
          }
        }
        __syncwarp();
      }
    });
  } else {
    // ---------------- epilogue (both CTAs: their 128 rows x TN) ----------------
    // one group per accumulator at most: two groups sharing one accumulator
    // barrier would wait on parities out of order
    constexpr int GROUPS = NACC < EPI_GROUPS ? NACC : EPI_GROUPS;
    const int q = warp & 3;
    const int grp = (warp - 6) / 4;
    const uint32_t stg_s = ptx::smem_u32(staging + (grp * 4 + q) * (32 * 33));
    const uint32_t acc_empty_leader = ptx::mapa(ptx::smem_u32(&acc_empty[0]), 0);
    int j = 0;
    for (int u = pair; u < units; u += pairs, ++j) {
      if ((j % GROUPS) != grp) continue;
      const Unit w = unit(u);
      const int a = j % NACC;
      ptx::mbar_wait(&acc_full[a], (j / NACC) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + a * G::ACC;
      float *part = ws + w.split * ws_split_stride;
      const int row0 = w.m0 + 128 * rank + 32 * q;
      if (SWAP && !(ACCT_SKIP(write_hi, 8))) {
        // lanes = output columns (this CTA's 128), TMEM columns = weight rows
        const int col = w.n0 + 128 * rank + 32 * q + lane;
        constexpr int CH = 16;
        for (int c = 0; c < TN / CH; ++c) {
          uint32_t r[CH];
          ptx::tmem_ld_32x32b_x16(trow + CH * c, r);
          if constexpr (DUAL) {
            uint32_t r2[CH];
            ptx::tmem_ld_32x32b_x16(trow + TN + CH * c, r2);
#pragma unroll
            for (int jj = 0; jj < CH; ++jj)
              r[jj] = __float_as_uint(__uint_as_float(r[jj]) + __uint_as_float(r2[jj]));
          }
          if (col >= N) continue;
          const int rbase = w.m0 + CH * c;
          if (splits == 1) {
            float cv[CH], bv[CH];
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) {
              const bool ok = rbase + jj < M;
              cv[jj] = (beta != 0.0f && ok) ? C[(int64_t)(rbase + jj) * ldc + col] : 0.0f;
              bv[jj] = (bias && ok) ? __ldg(bias + rbase + jj) : 0.0f;
            }
            float v[CH];
#pragma unroll
            for (int jj = 0; jj < CH; ++jj)
              v[jj] = finish_lin(__uint_as_float(r[jj]), alpha, beta, cv[jj], bias, bv[jj]);
            if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
            for (int jj = 0; jj < CH; ++jj)
              if (rbase + jj < M) C[(int64_t)(rbase + jj) * ldc + col] = v[jj];
          } else {
            float *dst = part + (int64_t)rbase * ws_ld + col;
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) __stcg(dst + (int64_t)jj * ws_ld, __uint_as_float(r[jj]));
          }
        }
      } else if (!(ACCT_SKIP(write_hi, 8))) {
        for (int c = 0; c < TN / 32; ++c) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(trow + 32 * c, r);
          if constexpr (DUAL) {
            uint32_t r2[32];
            ptx::tmem_ld_32x32b_x32(trow + TN + 32 * c, r2);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              r[jj] = __float_as_uint(__uint_as_float(r[jj]) + __uint_as_float(r2[jj]));
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) ptx::sts32(stg_s + 4 * (lane * 33 + jj), __uint_as_float(r[jj]));
          __syncwarp();
          const int col = w.n0 + 32 * c + lane;
          if (splits == 1) {
            const float my_bias = (bias && row0 + lane < M) ? __ldg(bias + row0 + lane) : 0.0f;
            float bv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) bv[i] = __shfl_sync(0xffffffffu, my_bias, i);
            if (col < N) {
              float cv[32];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                cv[i] = (beta != 0.0f && row0 + i < M) ? C[(int64_t)(row0 + i) * ldc + col] : 0.0f;
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                v[i] = finish_lin(ptx::lds32(stg_s + 4 * (i * 33 + lane)), alpha, beta, cv[i], bias,
                                  bv[i]);
              if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (row0 + i < M) C[(int64_t)(row0 + i) * ldc + col] = v[i];
            }
          } else {
            float *dst = part + (int64_t)row0 * ws_ld + col;
#pragma unroll 8
            for (int i = 0; i < 32; ++i)
              __stcg(dst + (int64_t)i * ws_ld, ptx::lds32(stg_s + 4 * (i * 33 + lane)));
          }
          __syncwarp();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(acc_empty_leader + 8 * a);
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // the leader's last MMAs (into both TMEMs) are drained
  if (warp == 1) ptx::tmem_dealloc2(tmem, 512);
}

// ------------------------------------------------ implicit-im2col conv (swap)
// 3x3 / stride 1 / pad 1 convolution as the swap-orientation tile
// (C^T = col^T . A^T: 128 output pixels x TN filters) WITHOUT the col array
// on the operand path -- the narrow layers (M <= 64) whose gemm is otherwise
// an HBM stream of col (yolov2-tiny layers 2 and 4: 24.9 and 12.5 MB per
// image) behind an im2col that writes it.
//
// A work unit is one image's TH x TW block of output pixels (TW = 16 or 8,
// TH = 128 / TW; MMA row m = a pixel of its warp's 8 x 4 block, conv_pixel).  Its input slab -- every
// channel's (TH + 2) x (TW + 2) window (stored TW + 8 wide from x0 - 4), one 4-D TMA box over (x, y, image,
// channel) whose out-of-bounds elements are zero, i.e. the conv's padding --
// makes every operand element one LDS at  lane base + immediate.
//   warp 0      TMA: all weight k-blocks once (resident, K-major SWIZZLE_128B),
//               then the slab of each unit through a ring of up to 8
// Two independent pipelines p = 0, 1 take alternate units (j = p, p + 2, ...):
//   warp 1 / 18 (TMEM allocator) + MMA issuer of pipeline p, exactly the swap
//               tile's 3xTF32 sequence (A = activations from TMEM, B = weights
//               hi / lo); two issuers because a narrow MMA is issue-bound
//   warps 2..5 / 6..9  weights lo once (all eight); then pipeline p's
//               activation operand: lane = pixel, k = (channel, kh, kw) ->
//               hi / lo to one of S TMEM stages; col of images >= col_from
//   warps 10..13 / 14..17  pipeline p's epilogue: tcgen05.ld -> beta C, bias
//               (staged in shared memory), leaky -> C, fused 2x2 maxpool
// Operand values, k order and MMA sequence equal im2col + the swap gemm, so
// C is bit-identical to the unfused pair (tests/test_gpu_kernels.py).
// MMA row m = 32 q + lane of a conv unit (TMEM lane quadrant q) <-> pixel:
// each warp holds an 8-wide x 4-tall block, so (1) its 32 slab addresses per
// tap, rows TWP = 24 floats apart, fall in 32 distinct banks (rows 0..3 at
// banks +0, +24, +16, +8) -- a 16 x 2 block had two lanes per bank on 8 of
// them -- and (2) it holds 4 x 2 whole 2x2 pooling windows
template <int TW>
__device__ __forceinline__ void conv_pixel(int q, int lane, int &py, int &px) {
  constexpr int BX = TW / 8;  // warp blocks per unit row
  px = 8 * (q % BX) + (lane & 7);
  py = 4 * (q / BX) + (lane >> 3);
}

template <int TN, int TW>
struct ConvCfg {
  static constexpr int BK = 32;
  // two independent MMA pipelines (alternate units, one issuing warp each):
  // a narrow 128 x TN x 8 MMA is bound by its issuing thread (~50 cycles at
  // N = 32, tools/mma_issue_probe.cu), not by the tensor core, so two issuers
  // double the SM's MMA rate.  Each pipeline owns 256 TMEM columns: NACC
  // accumulators of TN and S stages of the activation operand (hi, lo).
  // (TN = 32: 4 accumulators and 2 stages measured ~4% faster than 2 and 3;
  // each pipeline's accumulator barriers have ONE waiting group, in order)
  static constexpr int NP = 2, PCOLS = 256, NACC = TN <= 32 ? 4 : 2;
  static constexpr int S = (PCOLS - NACC * TN) / 64;
  static constexpr int TH = 128 / TW;
  // slab row: columns x0 - 4 .. x0 + TW + 3 (TMA needs a 16-byte aligned
  // start in the innermost dimension; a box starting at x0 - 1 faults)
  static constexpr int TWP = 24;  // >= TW + 6, and = 24 mod 32 (conv_pixel)
  static constexpr int SROWS = TH + 2;
  static constexpr int CS = SROWS * TWP * 4;      // slab bytes per channel
  static constexpr int W_TILE = TN * BK * 4;      // one weight k-block, K-major SW128
  static constexpr int A_COL0 = NACC * TN;          // within a pipeline's columns
  static constexpr int USED_COLS = NP * PCOLS;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t K_SBO = 8 * 128;
  static_assert(USED_COLS <= 512, "TMEM overflow");
};
constexpr int CONV_TC_THREADS = 32 * 26;  // wide conv: TMA, MMA, 16 builders, 8 epilogue
constexpr int kMaxSlabs = 8;  // slab ring depth: 2 .. 8 as shared memory allows
// warps: 0 TMA, 1 / 26 MMA issuers, 2-17 operand builders (two per TMEM lane
// quadrant and pipeline), 18-25 epilogue
constexpr int CONV_NARROW_THREADS = 32 * 27;

// One k-block (32 k = (channel, tap) pairs from k0 = 9 c0 + R0) of the
// activation operand for this lane's pixel: each k is one LDS at the lane's
// slab address (channel c0 folded in) plus a compile-time immediate -- the
// channel step and the tap's row / column offset.  TAIL: the last block of a
// K that is not a multiple of 32 (zeros past K).
// (K0, KEND: the part K0 .. KEND - 1 of the block, into v[K - K0] -- the
// narrow kernel's two operand warps per TMEM lane quadrant take 16 k each)
template <int TWP, int CS, int R0, int K, bool TAIL, int K0 = 0, int KEND = 32>
__device__ __forceinline__ void conv_ld(uint32_t base, int kvalid, float (&v)[KEND - K0]) {
  if constexpr (K < KEND) {
    constexpr int r = (R0 + K) % 9, dc = (R0 + K) / 9;
    constexpr int imm = dc * CS + ((r / 3) * TWP + r % 3 + 3) * 4;  // column x - 1 + kw
    if (TAIL && K >= kvalid)
      v[K - K0] = 0.0f;
    else
      asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v[K - K0]) : "r"(base), "n"(imm));
    conv_ld<TWP, CS, R0, K + 1, TAIL, K0, KEND>(base, kvalid, v);
  }
}

template <int TWP, int CS, int R0, int K0 = 0, int KEND = 32>
__device__ __forceinline__ void conv_block(uint32_t base, int kvalid, float (&v)[KEND - K0]) {
  if (kvalid >= KEND)
    conv_ld<TWP, CS, R0, K0, false, K0, KEND>(base, kvalid, v);
  else
    conv_ld<TWP, CS, R0, K0, true, K0, KEND>(base, kvalid, v);
}

// BETA: beta != 0 (C += ...) -- a template flag, so the usual beta = 0 launch
// issues no predicated C loads in the epilogue (as conv3x3_pool_kernel)
template <int TN, int TW, bool BETA>
__global__ void __launch_bounds__(CONV_NARROW_THREADS, 1)
tc_conv_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
               int M, int channels, int height, int width, int tiles_x, int tpi, int units,
               int nkb, float beta, float *__restrict__ C, int64_t ldc, int64_t c_bs,
               const float *__restrict__ bias, int act, float *__restrict__ col, int64_t ld_col,
               int64_t col_bs, int col_from, float *__restrict__ pool, int64_t ld_pool,
               int64_t pool_bs, int32_t *__restrict__ pidx, int64_t ld_pidx, int64_t pidx_bs,
               int c_from, int nslab, int dbg) {
  using G = ConvCfg<TN, TW>;
  constexpr int S = G::S, BK = G::BK, NACC = G::NACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *w_hi = base;                             // [nkb][W_TILE]
  uint8_t *w_lo = base + nkb * G::W_TILE;           // [nkb][W_TILE]
  const int slab_bytes = (channels * G::CS + 127) & ~127;
  uint8_t *slab0 = base + 2 * nkb * G::W_TILE;      // 2 x [channels][SROWS][TWP]
  uint64_t *wfull = reinterpret_cast<uint64_t *>(slab0 + nslab * slab_bytes);
  uint64_t *slab_full = wfull + 1;
  uint64_t *slab_empty = slab_full + kMaxSlabs;
  uint64_t *conv = slab_empty + kMaxSlabs;   // [NP][S]
  uint64_t *empty = conv + G::NP * S;         // [NP][S]
  uint64_t *acc_full = empty + G::NP * S;     // [NP][NACC]
  uint64_t *acc_empty = acc_full + G::NP * NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + G::NP * NACC);
  // 64 floats (16-B aligned: read as float4), then 8 x 8 x 33 scratch
  float *bias_s = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) &
                                            ~uintptr_t(15));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int HW = height * width;
  if (ACCT_TRACE(dbg) && blockIdx.x == 0 && threadIdx.x == 0) g_trace[6][0] = clock64();
  auto gtime = [] {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
  };
  if (ACCT_TRACE(dbg) && threadIdx.x == 0 && blockIdx.x < 256) g_trace[7][256 + blockIdx.x] = gtime();
  if (threadIdx.x == 0) {
    ptx::mbar_init(wfull, 1);
    for (int b = 0; b < nslab; ++b) {
      ptx::mbar_init(&slab_full[b], 1);
      ptx::mbar_init(&slab_empty[b], 8);  // the unit's pipeline's eight operand warps
    }
    for (int s = 0; s < G::NP * S; ++s) {
      ptx::mbar_init(&conv[s], 8);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < G::NP * NACC; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmW);
    ptx::prefetch_tmap(&tmX);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, G::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  const float inv_tpi = 1.0f / (float)tpi, inv_tx = 1.0f / (float)tiles_x;
  auto unit_xy = [&](int u, int &img, int &y0, int &x0) {
    int t, ty, tx;
    acct_divmod(u, tpi, inv_tpi, img, t);
    acct_divmod(t, tiles_x, inv_tx, ty, tx);
    y0 = ty * G::TH;
    x0 = tx * TW;
  };

  if (warp == 0) {
    // ---------------- TMA: resident weights, then the slabs ----------------
    if (lane == 0) {
      if (ACCT_SKIP(dbg, 16)) {
        ptx::mbar_arrive(wfull);
      } else {
        ptx::mbar_expect_tx(wfull, (uint32_t)(nkb * G::W_TILE));
        for (int kb = 0; kb < nkb; ++kb)
          ptx::tma_load_2d(w_hi + kb * G::W_TILE, &tmW, wfull, kb * BK, 0);
      }
      // slab ring position (sb, phase of its barriers) kept incrementally: no
      // runtime division per unit
      int j = 0, sb = 0, sph = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
        int img, y0, x0;
        unit_xy(u, img, y0, x0);
        if (j >= nslab) ptx::mbar_wait(&slab_empty[sb], sph ^ 1);
        if (ACCT_SKIP(dbg, 8)) {
          ptx::mbar_arrive(&slab_full[sb]);
        } else {
          ptx::mbar_expect_tx(&slab_full[sb], (uint32_t)(channels * G::CS));
          ptx::tma_load_4d(slab0 + sb * slab_bytes, &tmX, &slab_full[sb], x0 - 4, y0 - 1, img, 0);
        }
        if (++sb == nslab) {
          sb = 0;
          sph ^= 1;
        }
      }
    }
  } else if (warp == 1 || warp == 26) {
    // ---------------- MMA issuers: pipeline p takes units j = p, p + 2, ... ----------------
    const int p = warp == 26;
    constexpr uint32_t idesc = ptx::idesc_tf32(128, TN, false, false);
    const uint32_t pbase = tmem + p * G::PCOLS;
    int gp = 0, jp = 0;
    for (int u = blockIdx.x + p * gridDim.x; u < units; u += 2 * gridDim.x, ++jp) {
      const int a = jp % NACC;
      if (jp >= NACC) ptx::mbar_wait(&acc_empty[p * NACC + a], ((jp / NACC) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t d = pbase + a * TN;
      for (int kb = 0; kb < nkb; ++kb, ++gp) {
        const int s = gp % S;
        ptx::mbar_wait(&conv[p * S + s], (gp / S) & 1);
        if (ACCT_TRACE(dbg) && p == 0 && blockIdx.x == 0 && gp < kTrace && lane == 0) g_trace[2][gp] = clock64();
        ptx::tc_fence_after();
        const uint32_t yh = ptx::smem_u32(w_hi + kb * G::W_TILE);
        const uint32_t yl = ptx::smem_u32(w_lo + kb * G::W_TILE);
        const uint32_t at = pbase + G::A_COL0 + s * 2 * BK;
        // one elected lane issues the k-block's 12 MMAs and the stage commit
        if (ptx::elect_one()) {
          if (!(ACCT_SKIP(dbg, 2))) {
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t dyh = ptx::smem_desc(yh + 32 * k, 16, G::K_SBO, ptx::kLayoutSW128);
              const uint64_t dyl = ptx::smem_desc(yl + 32 * k, 16, G::K_SBO, ptx::kLayoutSW128);
              ptx::mma_tf32_ts(d, at + 8 * k, dyh, idesc, (kb | k) != 0);
              ptx::mma_tf32_ts(d, at + 8 * k, dyl, idesc, 1);
              ptx::mma_tf32_ts(d, at + BK + 8 * k, dyh, idesc, 1);
            }
          }
          ptx::mma_commit(&empty[p * S + s]);
        }
        __syncwarp();
        if (ACCT_TRACE(dbg) && p == 0 && blockIdx.x == 0 && gp < kTrace && lane == 0) g_trace[3][gp] = clock64();
      }
      if (ptx::elect_one()) ptx::mma_commit(&acc_full[p * NACC + a]);
      __syncwarp();
    }
  } else if (warp < 18) {
    // ---------------- weights lo, then the activation operand ----------------
    // two halves of eight warps (2-9, 10-17): half p builds every k-block of
    // its pipeline's units (j = p, p + 2, ...); within a half, the two warps
    // of a TMEM lane quadrant take k 0-15 and 16-31 of each block (four
    // warps, one per quadrant, were latency-bound: ~800 cycles per k-block)
    const int q = warp & 3;  // TMEM lanes 32q.. = MMA rows (pixels) 32q..
    const int half = (warp - 2) >> 3;
    const int kp = ((warp - 2) >> 2) & 1;
    const int ct = threadIdx.x - 64;
    const int K = 9 * channels;
    ptx::mbar_wait(wfull, 0);
    {
      const uint32_t hs = ptx::smem_u32(w_hi), ls = ptx::smem_u32(w_lo);
      for (int i = ct; i < nkb * G::W_TILE / 16; i += 512) {
        float4 h4;
        ptx::sts128(ls + 16 * i, split_lo(ptx::lds128(hs + 16 * i), h4));
      }
      ptx::fence_proxy_async_smem();
      // both halves wrote weights lo: all of it before any pipeline's first
      // conv arrival releases an MMA that reads it
      asm volatile("bar.sync 1, 512;" ::: "memory");
    }
    int py, px;
    conv_pixel<TW>(q, lane, py, px);
    const uint32_t lane_off = (uint32_t)((py * G::TWP + px) * 4);
    int g = 0, j = half;
    int sb = half % nslab, sph = half / nslab;  // slab ring position of unit j (j += 2)
    for (int u = blockIdx.x + half * gridDim.x; u < units; u += 2 * gridDim.x, j += 2) {
      int img, y0, x0;
      unit_xy(u, img, y0, x0);
      const int y = y0 + py, x = x0 + px;
      const bool wcol = img >= col_from;  // warp-uniform; lanes off the image skip the store
      const bool inside = y < height && x < width;
      float *colp = col + img * col_bs + (int64_t)y * width + x;
      const uint32_t lane_base = ptx::smem_u32(slab0 + sb * slab_bytes) + lane_off;
      if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && j < kTrace && ct % 128 == 0) g_trace[10][j] = clock64();
      ptx::mbar_wait(&slab_full[sb], sph & 1);
      if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && j < kTrace && ct % 128 == 0) g_trace[11][j] = clock64();
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S;
        const int k0 = kb * BK;
        const int c0 = k0 / 9;
        const int kvalid = K - k0;  // >= 32 except in the last block
        if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && g < kTrace && ct % 128 == 0) g_trace[0][g] = clock64();
        if (g >= S) ptx::mbar_wait(&empty[half * S + s], ((g / S) - 1) & 1);
        if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && g < kTrace && ct % 128 == 0) g_trace[1][g] = clock64();
        ptx::tc_fence_after();
        if (ACCT_SKIP(dbg, 1)) {  // profiling knob: skip building the operand (results wrong)
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&conv[half * S + s]);
          continue;
        }
        constexpr int KH = BK / 2;
        float v[KH];
        const uint32_t bc = lane_base + (uint32_t)(c0 * G::CS);
#define ACCT_CONV_PART(R0)                                                  \
  (kp ? conv_block<G::TWP, G::CS, R0, KH, BK>(bc, kvalid, v)                \
      : conv_block<G::TWP, G::CS, R0, 0, KH>(bc, kvalid, v))
        switch (k0 - 9 * c0) {
          case 0: ACCT_CONV_PART(0); break;
          case 1: ACCT_CONV_PART(1); break;
          case 2: ACCT_CONV_PART(2); break;
          case 3: ACCT_CONV_PART(3); break;
          case 4: ACCT_CONV_PART(4); break;
          case 5: ACCT_CONV_PART(5); break;
          case 6: ACCT_CONV_PART(6); break;
          case 7: ACCT_CONV_PART(7); break;
          default: ACCT_CONV_PART(8); break;
        }
#undef ACCT_CONV_PART
        if (wcol && inside) {
          const int kn = (kvalid < BK ? kvalid : BK) - KH * kp;
          float *cp = colp + (int64_t)(k0 + KH * kp) * ld_col;
#pragma unroll
          for (int k = 0; k < KH; ++k)
            if (k < kn) __stcs(cp + (int64_t)k * ld_col, v[k]);
        }
        uint32_t hi[KH], lo[KH];
#pragma unroll
        for (int k = 0; k < KH; ++k) {
          const uint32_t h = __float_as_uint(v[k]) & 0xFFFFE000u;
          hi[k] = h;
          lo[k] = __float_as_uint(v[k] - __uint_as_float(h));
        }
        if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && g < kTrace && ct % 128 == 0) g_trace[8][g] = clock64() + (lo[0] & 0);
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + half * G::PCOLS + G::A_COL0 +
                            s * 2 * BK + KH * kp;
        ptx::tmem_st_cols<KH>(ta, hi);
        ptx::tmem_st_cols<KH>(ta + BK, lo);
        ptx::tmem_st_wait();
        if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && g < kTrace && ct % 128 == 0) g_trace[9][g] = clock64();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&conv[half * S + s]);
        if (ACCT_TRACE(dbg) && half == 0 && blockIdx.x == 0 && g < kTrace && ct % 128 == 0) g_trace[4][g] = clock64();
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&slab_empty[sb]);  // this unit's slab is consumed
      sb += 2;
      while (sb >= nslab) {
        sb -= nslab;
        ++sph;
      }
    }
  } else {
    // ---------------- epilogue: lanes = pixels, TMEM columns = filters ----------------
    // group p of four warps (18-21, 22-25) drains pipeline p's accumulators
    const int q = warp & 3;
    const int grp = (warp - 18) >> 2;
    for (int i = threadIdx.x - 18 * 32; i < TN; i += 8 * 32) bias_s[i] = (bias && i < M) ? bias[i] : 0.0f;
    asm volatile("bar.sync 2, 256;" ::: "memory");  // the eight epilogue warps
    int py, px;
    conv_pixel<TW>(q, lane, py, px);
    // explicit shared-space addresses (generic LD/ST through the realigned
    // base measured several times slower): bias, this warp's pooling scratch
    const uint32_t bias_sa = ptx::smem_u32(bias_s);
    const uint32_t scr_sa = ptx::smem_u32(bias_s + 64 + (warp - 18) * 8 * 33);
    int jp = 0;
    for (int u = blockIdx.x + grp * gridDim.x; u < units; u += 2 * gridDim.x, ++jp) {
      int img, y0, x0;
      unit_xy(u, img, y0, x0);
      const int a = jp % NACC;
      ptx::mbar_wait(&acc_full[grp * NACC + a], (jp / NACC) & 1);
      if (ACCT_TRACE(dbg) && grp == 0 && blockIdx.x == 0 && jp < kTrace && lane == 0 && q == 0) g_trace[5][jp] = clock64();
      ptx::tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + grp * G::PCOLS + a * TN;
      const int y = y0 + py, x = x0 + px;
      const bool live = y < height && x < width && !(ACCT_SKIP(dbg, 4));
      const bool cst = live && img >= c_from;  // C of earlier images is dead when pooled here
      float *cp = C + img * c_bs + (int64_t)y * width + x;
      constexpr int CH = 16;
#pragma unroll 1
      for (int cc = 0; cc < TN / CH; ++cc) {
        uint32_t r[CH];
        if (ACCT_SKIP(dbg, 32)) continue;
        ptx::tmem_ld_32x32b_x16(trow + CH * cc, r);
        const int rbase = CH * cc;
        if (rbase >= M) continue;
        float *rp = cp + (int64_t)rbase * ldc;
        float cv[CH];
        if (BETA && live) {
#pragma unroll
          for (int jj = 0; jj < CH; ++jj)  // every load in flight before any store
            cv[jj] = rbase + jj < M ? rp[(int64_t)jj * ldc] : 0.0f;
        }
        float f[CH], bv[CH];
        if (bias) {
#pragma unroll
          for (int i4 = 0; i4 < CH / 4; ++i4) {
            const float4 b4 = ptx::lds128(bias_sa + 4 * (rbase + 4 * i4));
            bv[4 * i4] = b4.x; bv[4 * i4 + 1] = b4.y; bv[4 * i4 + 2] = b4.z; bv[4 * i4 + 3] = b4.w;
          }
        }
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) {
          float v = __uint_as_float(r[jj]);
          if (BETA && live) v = beta * cv[jj] + v;
          if (bias) v += bv[jj];
          f[jj] = v;
        }
        if (act == ACCT_ACT_LEAKY) acct_leaky_block(f);
        // C of the observable images only: a warp-uniform branch around the
        // stores (predicated per store they issued for every image)
        if (img >= c_from) {
#pragma unroll
          for (int jj = 0; jj < CH; ++jj)
            if (cst && rbase + jj < M) rp[(int64_t)jj * ldc] = f[jj];
        }
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) r[jj] = __float_as_uint(f[jj]);
#pragma unroll
        for (int half = 0; half < 2 && pool; ++half) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            ptx::sts32(scr_sa + 4 * (jj * 33 + lane), __uint_as_float(r[8 * half + jj]));
          // 2x2/2 maxpool, 8 filters per pass: the warp's 32 pixels are 8
          // whole windows (tiles start on even rows / columns); through the
          // scratch each lane takes window (lane & 7) of filters 4t + (lane >>
          // 3), comparing in darknet's scan order with strict '>' from -FLT_MAX
          __syncwarp();
          // window (lane & 7) of the warp's 8 x 4 block: top-left lane l0,
          // neighbours l0 + 1, + 8, + 9
          const int w8 = lane & 7, fg = lane >> 3;
          const int l0 = 16 * (w8 >> 2) + 2 * (w8 & 3);
          int wpy, wpx;
          conv_pixel<TW>(q, l0, wpy, wpx);
          const int wy = y0 + wpy, wx = x0 + wpx;
          const bool win = wy < height && wx < width && !(ACCT_SKIP(dbg, 4));
          const int64_t pofs = (int64_t)(wy >> 1) * (width >> 1) + (wx >> 1);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int fl = 4 * t + fg, f = rbase + 8 * half + fl;
            const uint32_t sv = scr_sa + 4 * (fl * 33 + l0);
            const float v00 = ptx::lds32(sv), v01 = ptx::lds32(sv + 4);
            const float v10 = ptx::lds32(sv + 4 * 8), v11 = ptx::lds32(sv + 4 * 9);
            if (win && f < M) {
              const int base_i = f * HW + wy * width + wx;
              float mx = -FLT_MAX;
              int32_t k = -1;
              if (v00 > mx) { mx = v00; k = base_i; }
              if (v01 > mx) { mx = v01; k = base_i + 1; }
              if (v10 > mx) { mx = v10; k = base_i + width; }
              if (v11 > mx) { mx = v11; k = base_i + width + 1; }
              pool[img * pool_bs + (int64_t)f * ld_pool + pofs] = mx;
              pidx[img * pidx_bs + (int64_t)f * ld_pidx + pofs] = k;
            }
          }
          __syncwarp();  // the scratch is rewritten by the next chunk
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[grp * NACC + a]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (ACCT_TRACE(dbg) && blockIdx.x == 0 && threadIdx.x == 0) g_trace[6][1] = clock64();
  if (ACCT_TRACE(dbg) && threadIdx.x == 0 && blockIdx.x < 256) g_trace[7][blockIdx.x] = gtime();
  if (warp == 1) ptx::tmem_dealloc(tmem, G::TMEM_COLS);
}

// ------------------------------------ implicit-im2col conv, wide layers
// The same fused conv for 128-filter blocks (M = 128 k, yolov2-tiny layers
// 6 and 8): weights no longer fit in shared memory, so each 32-deep k-block
// streams through a stage ring together with the slab CHUNK it reads -- the
// <= 5 input channels k0 / 9 .. (k0 + 31) / 9 of the unit's (TH+2) x (TW+2)
// window (one 4-D TMA box; channels past C read as zero).  A unit is one
// (128-filter block, image, TH x TW pixel block).  Swap orientation: MMA
// M = 128 pixels (TMEM lanes), N = 128 filters, 3xTF32 (A hi.W hi, A hi.W lo,
// A lo.W hi) per 8-deep k step.
//   warp 0      TMA: per stage the weight tile (128 rows x 32 k, SW128) and
//               the slab chunk
//   warp 1      TMEM allocator + MMA issuer
//   warps 2..17 two halves of eight taking alternate k-blocks: weights lo of
//               the stage, the activation operand (hi / lo to a TMEM stage;
//               two warps per lane quadrant, 16 k each), col of images >=
//               col_from
//   warps 18..25 epilogue, two groups taking alternate units (+ fused maxpool)
template <int TW>
struct WideCfg {
  static constexpr int TN = 128, BK = 32, S = 4, NACC = 2;  // NACC = 2: see the epilogue
  static constexpr int TH = 128 / TW;
  static constexpr int TWP = 24;  // >= TW + 6, and = 24 mod 32 (conv_pixel)
  static constexpr int SROWS = TH + 2;
  static constexpr int CS = SROWS * TWP * 4;      // slab bytes per channel
  static constexpr int CH_PER_KB = 5;             // channels a 32-deep k-block spans
  static constexpr int W_TILE = TN * BK * 4;      // 16 KB
  static constexpr int SLAB = ((CH_PER_KB * CS) + 1023) & ~1023;
  static constexpr int STAGE = 2 * W_TILE + SLAB; // W hi, W lo, slab chunk
  static constexpr int A_COL0 = NACC * TN;
  static constexpr int USED_COLS = NACC * TN + S * 2 * BK;
  static constexpr uint32_t K_SBO = 8 * 128;
  static_assert(USED_COLS <= 512, "TMEM overflow");
};

template <int TW, bool BETA>
__global__ void __launch_bounds__(CONV_TC_THREADS, 1)
tc_conv_wide_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    int M, int channels, int height, int width, int tiles_x, int tpi, int units,
                    int nkb, float beta, float *__restrict__ C, int64_t ldc, int64_t c_bs,
                    const float *__restrict__ bias, int act, float *__restrict__ col,
                    int64_t ld_col, int64_t col_bs, int col_from, float *__restrict__ pool,
                    int64_t ld_pool, int64_t pool_bs, int32_t *__restrict__ pidx, int64_t ld_pidx,
                    int64_t pidx_bs, int c_from, int batch, int dbg) {
  using G = WideCfg<TW>;
  constexpr int S = G::S, BK = G::BK, NACC = G::NACC, TN = G::TN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  auto w_hi = [&](int s) { return base + s * G::STAGE; };
  auto w_lo = [&](int s) { return base + s * G::STAGE + G::W_TILE; };
  auto slab = [&](int s) { return base + s * G::STAGE + 2 * G::W_TILE; };
  uint64_t *full = reinterpret_cast<uint64_t *>(base + S * G::STAGE);
  uint64_t *conv = full + S;
  uint64_t *empty = conv + S;
  uint64_t *acc_full = empty + S;
  uint64_t *acc_empty = acc_full + NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + NACC);
  // all M <= 256 biases (16-B aligned: read as float4), then 8 x 8 x 33 scratch
  float *bias_s = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) &
                                            ~uintptr_t(15));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int HW = height * width;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 8);   // the k-block's group of eight builder warps
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmW);
    ptx::prefetch_tmap(&tmX);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  const int per_mb = tpi * batch;
  const float inv_mb = 1.0f / (float)per_mb, inv_tpi = 1.0f / (float)tpi,
              inv_tx = 1.0f / (float)tiles_x;
  auto unit_of = [&](int u, int &mb, int &img, int &y0, int &x0) {
    int r, t, ty, tx;
    acct_divmod(u, per_mb, inv_mb, mb, r);
    acct_divmod(r, tpi, inv_tpi, img, t);
    acct_divmod(t, tiles_x, inv_tx, ty, tx);
    y0 = ty * G::TH;
    x0 = tx * TW;
  };

  if (warp == 0) {
    // ---------------- TMA: weight tile + slab chunk per stage ----------------
    if (lane == 0) {
      int g = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mb, img, y0, x0;
        unit_of(u, mb, img, y0, x0);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          if (g >= S) ptx::mbar_wait(&empty[s], ((g / S) - 1) & 1);
          // dbg 8 / 16: skip the weight / slab load (pipeline analysis only)
          ptx::mbar_expect_tx(&full[s], (uint32_t)((ACCT_SKIP(dbg, 8) ? 0 : G::W_TILE) +
                                                   (ACCT_SKIP(dbg, 16) ? 0 : G::CH_PER_KB * G::CS)));
          if (!(ACCT_SKIP(dbg, 8))) ptx::tma_load_2d(w_hi(s), &tmW, &full[s], kb * BK, mb * TN);
          if (!(ACCT_SKIP(dbg, 16)))
            ptx::tma_load_4d(slab(s), &tmX, &full[s], x0 - 4, y0 - 1, img, (kb * BK) / 9);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = ptx::idesc_tf32(128, TN, false, false);
    int g = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int a = j % NACC;
      if (j >= NACC) ptx::mbar_wait(&acc_empty[a], ((j / NACC) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem + a * TN;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S;
        ptx::mbar_wait(&conv[s], (g / S) & 1);
        ptx::tc_fence_after();
        const uint32_t yh = ptx::smem_u32(w_hi(s)), yl = ptx::smem_u32(w_lo(s));
        const uint32_t at = tmem + G::A_COL0 + s * 2 * BK;
        if (ptx::elect_one()) {
          if (!(ACCT_SKIP(dbg, 2))) {
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t dyh = ptx::smem_desc(yh + 32 * k, 16, G::K_SBO, ptx::kLayoutSW128);
              const uint64_t dyl = ptx::smem_desc(yl + 32 * k, 16, G::K_SBO, ptx::kLayoutSW128);
              ptx::mma_tf32_ts(d, at + 8 * k, dyh, idesc, (kb | k) != 0);
              ptx::mma_tf32_ts(d, at + 8 * k, dyl, idesc, 1);
              ptx::mma_tf32_ts(d, at + BK + 8 * k, dyh, idesc, 1);
            }
          }
          ptx::mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma_commit(&acc_full[a]);
      __syncwarp();
    }
  } else if (warp < 18) {
    // ---------------- weights lo + activation operand (two halves) ----------------
    // half h (warps 2-9, 10-17) takes k-blocks g = h mod 2; within a half
    // the two warps of a TMEM lane quadrant take k 0-15 and 16-31 (one warp
    // per quadrant was latency-bound, as in the narrow conv)
    const int q = warp & 3;
    const int half = (warp - 2) >> 3;
    const int kp = ((warp - 2) >> 2) & 1;
    const int ht = threadIdx.x - 64 - 256 * half;  // 0..255 within the half
    const int K = 9 * channels;
    int py, px;
    conv_pixel<TW>(q, lane, py, px);
    const uint32_t lane_off = (uint32_t)((py * G::TWP + px) * 4);
    int g = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int mb, img, y0, x0;
      unit_of(u, mb, img, y0, x0);
      const int y = y0 + py, x = x0 + px;
      const bool wcol = img >= col_from && mb == 0;  // col once, by the first filter block
      const bool inside = y < height && x < width;
      float *colp = col + img * col_bs + (int64_t)y * width + x;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        if ((g & 1) != half) continue;
        const int s = g % S;
        const int k0 = kb * BK;
        const int kvalid = K - k0;
        ptx::mbar_wait(&full[s], (g / S) & 1);
        if (!(ACCT_SKIP(dbg, 1))) {
          // weights lo of this stage (this half's 128 threads)
          const uint32_t hs = ptx::smem_u32(w_hi(s)), ls = ptx::smem_u32(w_lo(s));
#pragma unroll
          for (int i = 0; i < G::W_TILE / 16 / 256; ++i) {
            float4 h4;
            const uint32_t o = 16 * (ht + 256 * i);
            ptx::sts128(ls + o, split_lo(ptx::lds128(hs + o), h4));
          }
          constexpr int KH = BK / 2;
          float v[KH];
          const uint32_t bc = ptx::smem_u32(slab(s)) + lane_off;  // chunk starts at channel k0 / 9
#define ACCT_CONV_PART(R0)                                                  \
  (kp ? conv_block<G::TWP, G::CS, R0, KH, BK>(bc, kvalid, v)                \
      : conv_block<G::TWP, G::CS, R0, 0, KH>(bc, kvalid, v))
          switch (k0 % 9) {
            case 0: ACCT_CONV_PART(0); break;
            case 1: ACCT_CONV_PART(1); break;
            case 2: ACCT_CONV_PART(2); break;
            case 3: ACCT_CONV_PART(3); break;
            case 4: ACCT_CONV_PART(4); break;
            case 5: ACCT_CONV_PART(5); break;
            case 6: ACCT_CONV_PART(6); break;
            case 7: ACCT_CONV_PART(7); break;
            default: ACCT_CONV_PART(8); break;
          }
#undef ACCT_CONV_PART
          if (wcol && inside) {
            const int kn = (kvalid < BK ? kvalid : BK) - KH * kp;
            float *cp = colp + (int64_t)(k0 + KH * kp) * ld_col;
#pragma unroll
            for (int k = 0; k < KH; ++k)
              if (k < kn) __stcs(cp + (int64_t)k * ld_col, v[k]);
          }
          uint32_t hi[KH], lo[KH];
#pragma unroll
          for (int k = 0; k < KH; ++k) {
            const uint32_t h = __float_as_uint(v[k]) & 0xFFFFE000u;
            hi[k] = h;
            lo[k] = __float_as_uint(v[k] - __uint_as_float(h));
          }
          const uint32_t ta =
              tmem + ((uint32_t)(32 * q) << 16) + G::A_COL0 + s * 2 * BK + KH * kp;
          ptx::tmem_st_cols<KH>(ta, hi);
          ptx::tmem_st_cols<KH>(ta + BK, lo);
          ptx::tmem_st_wait();
          ptx::fence_proxy_async_smem();  // weights lo -> the tensor core
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ---------------- epilogue: two groups taking alternate units ----------------
    // (safe with NACC = 2 only: group g always drains accumulator g, so each
    // acc barrier has one waiter; one accumulator with alternating groups
    // would interleave parities on one barrier -- measured wrong on yolov2-608)
    const int q = warp & 3;
    const int grp = (warp - 18) >> 2;
    int py, px;
    conv_pixel<TW>(q, lane, py, px);
    for (int i = threadIdx.x - 18 * 32; i < 256; i += 8 * 32) bias_s[i] = (bias && i < M) ? bias[i] : 0.0f;
    asm volatile("bar.sync 2, 256;" ::: "memory");  // the eight epilogue warps
    const uint32_t bias_sa = ptx::smem_u32(bias_s);
    const uint32_t scr_sa = ptx::smem_u32(bias_s + 256 + (warp - 18) * 8 * 33);
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      if ((j & 1) != grp) continue;
      int mb, img, y0, x0;
      unit_of(u, mb, img, y0, x0);
      const int a = j % NACC;
      ptx::mbar_wait(&acc_full[a], (j / NACC) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + a * TN;
      const int y = y0 + py, x = x0 + px;
      const bool live = y < height && x < width && !(ACCT_SKIP(dbg, 4));
      const bool cst = live && img >= c_from;
      const int m0 = mb * TN;  // this unit's first filter
      float *cp = C + img * c_bs + (int64_t)y * width + x;
      constexpr int CH = 16;
#pragma unroll 1
      for (int cc = 0; cc < TN / CH; ++cc) {
        uint32_t r[CH];
        ptx::tmem_ld_32x32b_x16(trow + CH * cc, r);
        const int rbase = m0 + CH * cc;
        if (rbase >= M) continue;
        float *rp = cp + (int64_t)rbase * ldc;
        float cv[CH];
        if (BETA && live) {
#pragma unroll
          for (int jj = 0; jj < CH; ++jj) cv[jj] = rbase + jj < M ? rp[(int64_t)jj * ldc] : 0.0f;
        }
        float f[CH], bv[CH];
        if (bias) {
#pragma unroll
          for (int i4 = 0; i4 < CH / 4; ++i4) {
            const float4 b4 = ptx::lds128(bias_sa + 4 * (rbase + 4 * i4));
            bv[4 * i4] = b4.x; bv[4 * i4 + 1] = b4.y; bv[4 * i4 + 2] = b4.z; bv[4 * i4 + 3] = b4.w;
          }
        }
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) {
          float v = __uint_as_float(r[jj]);
          if (BETA && live) v = beta * cv[jj] + v;
          if (bias) v += bv[jj];
          f[jj] = v;
        }
        if (act == ACCT_ACT_LEAKY) acct_leaky_block(f);
        // C of the observable images only: a warp-uniform branch around the
        // stores (predicated per store they issued for every image)
        if (img >= c_from) {
#pragma unroll
          for (int jj = 0; jj < CH; ++jj)
            if (cst && rbase + jj < M) rp[(int64_t)jj * ldc] = f[jj];
        }
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) r[jj] = __float_as_uint(f[jj]);
#pragma unroll
        for (int hf = 0; hf < 2 && pool; ++hf) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            ptx::sts32(scr_sa + 4 * (jj * 33 + lane), __uint_as_float(r[8 * hf + jj]));
          __syncwarp();
          const int w8 = lane & 7, fg = lane >> 3;
          const int l0 = 16 * (w8 >> 2) + 2 * (w8 & 3);
          int wpy, wpx;
          conv_pixel<TW>(q, l0, wpy, wpx);
          const int wy = y0 + wpy, wx = x0 + wpx;
          const bool win = wy < height && wx < width && !(ACCT_SKIP(dbg, 4));
          const int64_t pofs = (int64_t)(wy >> 1) * (width >> 1) + (wx >> 1);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int fl = 4 * t + fg, f = rbase + 8 * hf + fl;
            const uint32_t sv = scr_sa + 4 * (fl * 33 + l0);
            const float v00 = ptx::lds32(sv), v01 = ptx::lds32(sv + 4);
            const float v10 = ptx::lds32(sv + 4 * 8), v11 = ptx::lds32(sv + 4 * 9);
            if (win && f < M) {
              const int base_i = f * HW + wy * width + wx;
              float mx = -FLT_MAX;
              int32_t k = -1;
              if (v00 > mx) { mx = v00; k = base_i; }
              if (v01 > mx) { mx = v01; k = base_i + 1; }
              if (v10 > mx) { mx = v10; k = base_i + width; }
              if (v11 > mx) { mx = v11; k = base_i + width + 1; }
              pool[img * pool_bs + (int64_t)f * ld_pool + pofs] = mx;
              pidx[img * pidx_bs + (int64_t)f * ld_pidx + pofs] = k;
            }
          }
          __syncwarp();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[a]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------ row-band conv (narrow layers)
// 3x3 / stride 1 / pad 1 convolution of M <= 64 filters as shifted MMAs: no
// im2col operand is built at all.  A work unit is one image's output row
// PAIR (2P, 2P + 1) over a column strip x0 .. x0 + wdt - 1 (wdt <= 128): MMA
// row i = output column x0 + i, N = filters.  The input rows 2P - 1 .. 2P + 2
// of 8 channels at a time are staged in shared memory channel-quad-major,
// position-major -- [row][quad][position][4 channels], one 16-B row per
// position, the no-swizzle K-major canonical layout -- so the operand of tap
// (kh, kw) for output row 2P + a is the SAME bytes read through a descriptor
// whose start is (a + kh) rows and kw positions further (tools/nosw_probe.cu
// checks the layout and the 16-B shifts).  Each input value is staged (and
// split) once per 8-channel step instead of once per tap.
// 3xTF32 in two MMAs per (tap, 8 channels): A hi x [W hi | W lo] (N = 2 TN)
// and A lo x W hi (N = TN) into the first half; the epilogue adds the halves.
// tcgen05 reads both shared-memory operands at ~128 B/clk (tools/nosw_probe:
// a 128 x 32 x 8 ss MMA costs 40 cycles per SM whatever the issuers), so two
// MMAs instead of three: 88 rather than 120 cycles per step at TN = 32.
//   warps 0-7  stage (LDG, hi/lo split, STS) through a ring of nstage steps:
//              two groups of four taking alternate steps, all of a step's
//              loads in flight at once (one group alone was latency-bound)
//   warps 8, 9 MMA issuers: warp 8 + a fills output row 2P + a; with the
//              epilogue warps they split the weights into shared memory
//              while the first steps are staged
//   warps 10-17 epilogue, two groups of four taking alternate units (one
//              warp per TMEM lane quadrant was latency-bound): tcgen05.ld
//              (lane = column), + bias, leaky -> C, and the fused 2x2 maxpool
//              (vertical in-thread, horizontal by one lane exchange; two
//              filters per store)
// Not bit-identical to im2col + the gemm (another summation order); within
// the gemm tolerance of the oracle (tests/test_gpu_kernels.py).
template <int TN>
struct RowsCfg {
  static constexpr int UCOLS = 4 * TN;             // a unit: 2 rows x [main | lo] x TN
  static constexpr int NACC = 512 / UCOLS;         // units in flight (TMEM)
  static constexpr int MAXS = 8;                   // staging ring depth
};
constexpr int ROWS_THREADS = 32 * 18;
constexpr int ROWS_ITEMS = (8 * 130 + 127) / 128;  // staged positions per thread and step

// The weights' shared-memory image, once per launch: [tap][8-channel step]
// [quad][2 TN rows][4 channels] with W hi in rows 0..TN-1 and W lo in rows
// TN..2TN-1 (zero rows past M); every CTA of the conv bulk-copies it.
template <int TN>
__global__ void __launch_bounds__(256)
rows_weights_kernel(const float *__restrict__ A, int64_t lda, int M, int channels,
                    float4 *__restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int nq = channels / 4, items = 9 * nq * TN;
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= items) return;
  const int n = i % TN, r = i / TN;  // r = tap * nq + cq
  const int tap = r / nq, cq = r - tap * nq;
  float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (n < M) {
    const float *p = A + (int64_t)n * lda + 36 * cq + tap;
    v = make_float4(p[0], p[9], p[18], p[27]);
  }
  float4 h;
  const float4 l = split_lo(v, h);
  const int row0 = ((tap * (nq / 2) + (cq >> 1)) * 2 + (cq & 1)) * 2 * TN;
  out[row0 + n] = h;
  out[row0 + TN + n] = l;
}

template <int TN>
__global__ void __launch_bounds__(ROWS_THREADS, 1)
tc_conv_rows_kernel(const float *__restrict__ im, int64_t ld_im, int64_t im_bs, int channels,
                    int height, int width, const float4 *__restrict__ wimg, int M,
                    float *__restrict__ col, int64_t ld_col, int64_t col_bs, int col_from,
                    int nstrips, int swd, int sp, int pairs, int units, int nstage, float beta,
                    float *__restrict__ C, int64_t ldc, int64_t c_bs,
                    const float *__restrict__ bias, int act, float *__restrict__ pool,
                    int64_t ld_pool, int64_t pool_bs, int32_t *__restrict__ pidx,
                    int64_t ld_pidx, int64_t pidx_bs, int c_from, int dbg) {
  using G = RowsCfg<TN>;
  constexpr int NACC = G::NACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int stage_bytes = 256 * sp;                 // hi then lo: 4 rows x 2 quads x sp x 16 B
  uint8_t *stages = base;
  uint8_t *wts = base + nstage * stage_bytes;       // [tap][step][quad][2 TN][4]
  const int nsteps = channels / 8;
  const int w_bytes = 9 * nsteps * 2 * 2 * TN * 16;
  float *bias_s = reinterpret_cast<float *>(wts + w_bytes);
  uint64_t *slab_full = reinterpret_cast<uint64_t *>(bias_s + TN);
  uint64_t *slab_empty = slab_full + G::MAXS;
  uint64_t *acc_full = slab_empty + G::MAXS;
  uint64_t *acc_empty = acc_full + NACC;
  uint64_t *wfull = acc_empty + NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(wfull, 1);
    for (int s = 0; s < nstage; ++s) {
      ptx::mbar_init(&slab_full[s], 4);   // the four staging warps
      ptx::mbar_init(&slab_empty[s], 2);  // both issuers' commits
    }
    for (int a = 0; a < NACC; ++a) {
      ptx::mbar_init(&acc_full[a], 2);
      ptx::mbar_init(&acc_empty[a], 4);   // the four epilogue warps
    }
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 32 * 8) {
    // the weights, already in their shared-memory image (rows_weights_kernel),
    // by bulk copies of <= 64 KB
    ptx::mbar_expect_tx(wfull, (uint32_t)w_bytes);
    for (int o = 0; o < w_bytes; o += 65536)
      ptx::bulk_load(wts + o, reinterpret_cast<const uint8_t *>(wimg) + o,
                     (uint32_t)min(65536, w_bytes - o), wfull);
  }
  if (warp >= 10) {
    for (int i = threadIdx.x - 320; i < TN; i += 256) bias_s[i] = (bias && i < M) ? bias[i] : 0.0f;
    asm volatile("bar.sync 1, 256;" ::: "memory");  // the epilogue warps: bias written
  }
  const int per_img = nstrips * pairs;
  auto unit_of = [&](int u, int &img, int &x0, int &wdt, int &y0) {
    img = u / per_img;
    const int r = u - img * per_img;
    const int strip = r / pairs;
    y0 = 2 * (r - strip * pairs);
    x0 = strip * swd;
    wdt = min(swd, width - x0);
  };

  if (warp < 8) {
    // ---------------- staging: 4 input rows x 8 channels per step ----------------
    const int grp = warp >> 2, t = threadIdx.x & 127;
    int s = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int img, x0, wdt, y0;
      unit_of(u, img, x0, wdt, y0);
      const float *src = im + img * im_bs;
      for (int g = 0; g < nsteps; ++g, ++s) {
        if ((s & 1) != grp) continue;
        const int st = s % nstage;
        if (s >= nstage) ptx::mbar_wait(&slab_empty[st], ((s / nstage) - 1) & 1);
        if (ACCT_SKIP(dbg, 8)) {  // profiling: no staging at all
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&slab_full[st]);
          continue;
        }
        const uint32_t hb = ptx::smem_u32(stages + st * stage_bytes);
        const uint32_t lb = hb + 128 * sp;
        const float *cs = src + (int64_t)(8 * g) * ld_im;
        // every load of the step in flight before the first use (a loop of
        // load -> split -> store per item was latency-bound: ~8k cycles/step)
        float4 v[ROWS_ITEMS];
#pragma unroll
        for (int it = 0; it < ROWS_ITEMS; ++it) {
          const int i = t + 128 * it;
          const int rq = i / sp, pos = i - rq * sp;  // rq = row * 2 + quad
          const int y = y0 - 1 + (rq >> 1), x = x0 - 1 + pos;
          v[it] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (i < 8 * sp && y >= 0 && y < height && x >= 0 && x < width && pos <= wdt + 1 &&
              !ACCT_SKIP(dbg, 1)) {
            const float *p = cs + (int64_t)(4 * (rq & 1)) * ld_im + (int64_t)y * width + x;
            v[it].x = __ldg(p);
            v[it].y = __ldg(p + ld_im);
            v[it].z = __ldg(p + 2 * ld_im);
            v[it].w = __ldg(p + 3 * ld_im);
          }
        }
#pragma unroll
        for (int it = 0; it < ROWS_ITEMS; ++it) {
          const int i = t + 128 * it;
          if (i < 8 * sp) {
            float4 h;
            const float4 l = split_lo(v[it], h);
            ptx::sts128(hb + 16 * i, h);
            ptx::sts128(lb + 16 * i, l);
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&slab_full[st]);
        if (col && img >= col_from) {
          // col of an observable image from the same registers: input (y, x)
          // of channel c is col row 9 c + 3 kh + kw at output (y + 1 - kh,
          // x + 1 - kw) for the unit's two rows and strip (each col element
          // once; zero padding included)
          float *cb = col + img * col_bs;
#pragma unroll
          for (int it = 0; it < ROWS_ITEMS; ++it) {
            const int i = t + 128 * it;
            if (i >= 8 * sp) continue;
            const int rq = i / sp, pos = i - rq * sp;
            const int yi = y0 - 1 + (rq >> 1), xi = x0 - 1 + pos;
            const int c0 = 8 * g + 4 * (rq & 1);
            const float vv[4] = {v[it].x, v[it].y, v[it].z, v[it].w};
#pragma unroll
            for (int kh = 0; kh < 3; ++kh) {
              const int yo = yi + 1 - kh;
              if (yo < y0 || yo > y0 + 1 || yo >= height) continue;
#pragma unroll
              for (int kw = 0; kw < 3; ++kw) {
                const int xo = xi + 1 - kw;
                if (xo < x0 || xo >= x0 + wdt) continue;
                float *cp = cb + (int64_t)(9 * c0 + 3 * kh + kw) * ld_col + (int64_t)yo * width + xo;
#pragma unroll
                for (int e = 0; e < 4; ++e) __stcs(cp + (int64_t)(9 * e) * ld_col, vv[e]);
              }
            }
          }
        }
      }
    }
  } else if (warp < 10) {
    // ---------------- MMA issuers: warp 8 + a -> output row 2P + a ----------------
    const int a = warp - 8;
    constexpr uint32_t idesc_w = ptx::idesc_tf32(128, 2 * TN, false, false);
    constexpr uint32_t idesc_h = ptx::idesc_tf32(128, TN, false, false);
    const uint32_t st0 = ptx::smem_u32(stages), w0 = ptx::smem_u32(wts);
    ptx::mbar_wait(wfull, 0);
    int s = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int slot = j % NACC;
      if (j >= NACC) ptx::mbar_wait(&acc_empty[slot], ((j / NACC) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem + slot * G::UCOLS + a * 2 * TN;
      for (int g = 0; g < nsteps; ++g, ++s) {
        const int st = s % nstage;
        ptx::mbar_wait(&slab_full[st], (s / nstage) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t hb = st0 + st * stage_bytes;
#pragma unroll
          for (int tap = 0; tap < 9 && !ACCT_SKIP(dbg, 2); ++tap) {
            const int kh = tap / 3, kw = tap % 3;
            const uint32_t ao = (uint32_t)((a + kh) * 2 * sp + kw) * 16;
            const uint64_t ah = ptx::smem_desc(hb + ao, sp * 16, 128, 0);
            const uint64_t al = ptx::smem_desc(hb + 128 * sp + ao, sp * 16, 128, 0);
            const uint64_t bw = ptx::smem_desc(w0 + (uint32_t)((tap * nsteps + g) * 2) * 2 * TN * 16,
                                               2 * TN * 16, 128, 0);
            ptx::mma_tf32(d, ah, bw, idesc_w, (g | tap) != 0);
            ptx::mma_tf32(d, al, bw, idesc_h, 1);
          }
          ptx::mma_commit(&slab_empty[st]);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma_commit(&acc_full[slot]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: lane = output column, TMEM columns = filters ----------------
    const int q = warp & 3, eg = (warp - 10) >> 2;
    const int HW = height * width;
    const unsigned full = 0xffffffffu;
    const bool odd = lane & 1;
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      if ((j & 1) != eg) continue;
      int img, x0, wdt, y0;
      unit_of(u, img, x0, wdt, y0);
      const int slot = j % NACC;
      ptx::mbar_wait(&acc_full[slot], (j / NACC) & 1);
      ptx::tc_fence_after();
      const int xl = 32 * q + lane, x = x0 + xl;
      const bool live = xl < wdt;
      const bool row1 = y0 + 1 < height;
      const bool cst = live && img >= c_from;
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + slot * G::UCOLS;
      float *cp = C + img * c_bs + (int64_t)y0 * width + x;
      if (ACCT_SKIP(dbg, 4)) {  // profiling: no epilogue work
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&acc_empty[slot]);
        continue;
      }
      const int xe = x & ~1;  // this lane's pooling window (even column)
      const bool wlive = (xl & ~1) < wdt;
      const int64_t pofs = (int64_t)(y0 >> 1) * (width >> 1) + (xe >> 1);
#pragma unroll 1
      for (int cc = 0; cc < TN / 16; ++cc) {
        uint32_t m0[16], l0[16], m1[16], l1[16];
        ptx::tmem_ld_32x32b_x16_nw(trow + 16 * cc, m0);
        ptx::tmem_ld_32x32b_x16_nw(trow + TN + 16 * cc, l0);
        ptx::tmem_ld_32x32b_x16_nw(trow + 2 * TN + 16 * cc, m1);
        ptx::tmem_ld_32x32b_x16_nw(trow + 3 * TN + 16 * cc, l1);
        ptx::tmem_ld_wait();
        const int f0 = 16 * cc;
        if (f0 >= M) continue;
        float v0[16], v1[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v0[i] = __uint_as_float(m0[i]) + __uint_as_float(l0[i]);
          v1[i] = __uint_as_float(m1[i]) + __uint_as_float(l1[i]);
        }
        if (beta != 0.0f && live) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (f0 + i < M) {
              v0[i] = beta * cp[(int64_t)(f0 + i) * ldc] + v0[i];
              if (row1) v1[i] = beta * cp[(int64_t)(f0 + i) * ldc + width] + v1[i];
            }
          }
        }
        if (bias) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float b = bias_s[f0 + i];
            v0[i] += b;
            v1[i] += b;
          }
        }
        if (act == ACCT_ACT_LEAKY) {
          acct_leaky_block(v0);
          acct_leaky_block(v1);
        }
        if (cst) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (f0 + i < M) {
              cp[(int64_t)(f0 + i) * ldc] = v0[i];
              if (row1) cp[(int64_t)(f0 + i) * ldc + width] = v1[i];
            }
          }
        }
        if (pool) {
          // window of filter f0 + i + odd at (y0, xe): even lanes own column
          // xe, odd lanes xe + 1; one exchange gives each lane its partner's
          // pair of the filter it pools
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float r0 = __shfl_xor_sync(full, odd ? v0[i] : v0[i + 1], 1);
            const float r1 = __shfl_xor_sync(full, odd ? v1[i] : v1[i + 1], 1);
            const float p00 = odd ? r0 : v0[i], p01 = odd ? v0[i + 1] : r0;
            const float p10 = odd ? r1 : v1[i], p11 = odd ? v1[i + 1] : r1;
            const int f = f0 + i + (odd ? 1 : 0);
            if (wlive && f < M) {
              const int bi = f * HW + y0 * width + xe;
              float mx = -FLT_MAX;
              int32_t k = -1;
              if (p00 > mx) { mx = p00; k = bi; }
              if (p01 > mx) { mx = p01; k = bi + 1; }
              if (p10 > mx) { mx = p10; k = bi + width; }
              if (p11 > mx) { mx = p11; k = bi + width + 1; }
              pool[img * pool_bs + (int64_t)f * ld_pool + pofs] = mx;
              pidx[img * pidx_bs + (int64_t)f * ld_pidx + pofs] = k;
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[slot]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) ptx::tmem_dealloc(tmem, 512);
}

// Sum the split-K partials of every output element in split order and apply
// the epilogue (grid-wide, one thread per 4 consecutive columns).
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const float *__restrict__ ws, int64_t ws_ld, int64_t split_stride, int splits,
                     int M, int N, float alpha, float beta, float *__restrict__ C, int64_t ldc,
                     const float *__restrict__ bias, int act) {
  pdl_trigger();
  pdl_wait();
  const int nq = (N + 3) / 4;
  const int total = M * nq;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int row = t / nq;
    const int col = (t - row * nq) * 4;
    const float *p = ws + (int64_t)row * ws_ld + col;
    float4 acc = __ldcg(reinterpret_cast<const float4 *>(p));
    for (int sp = 1; sp < splits; ++sp) {
      const float4 v = __ldcg(reinterpret_cast<const float4 *>(p + sp * split_stride));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const float bv = bias ? __ldg(bias + row) : 0.0f;
    float *cp = C + (int64_t)row * ldc + col;
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = finish_lin(a4[e], alpha, beta, beta != 0.0f && col + e < N ? cp[e] : 0.0f, bias, bv);
    if (act == ACCT_ACT_LEAKY) acct_leaky_block(v);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (col + e < N) cp[e] = v[e];
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D fp32 tensor map: inner dim `inner` (contiguous), outer dim `outer` with
// row pitch `ld` elements; box = box_inner x box_outer; out-of-bounds reads are 0.
bool make_map(CUtensorMap *map, const float *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor maps are pure functions of (pointer, shape, pitch, box, swizzle);
// the executor replays the same few dozen per image, so encode each once per
// host thread.
struct MapKey {
  const void *ptr;
  uint64_t inner, outer, ld;
  uint32_t box, box_in, swz;
  bool operator==(const MapKey &o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && box == o.box &&
           box_in == o.box_in && swz == o.swz;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey &k) const {
    uint64_t h = reinterpret_cast<uint64_t>(k.ptr) * 0x9E3779B97F4A7C15ull;
    h ^= k.inner + 0x9E37 + (h << 6) + (h >> 2);
    h ^= k.outer + 0x7F4A + (h << 6) + (h >> 2);
    h ^= k.ld + ((uint64_t)k.box << 32) + ((uint64_t)k.swz << 48) + ((uint64_t)k.box_in << 56) +
         (h << 6) + (h >> 2);
    return (size_t)h;
  }
};

bool cached_map(CUtensorMap *map, const float *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  static thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, inner, outer, ld, box_outer, box_inner, (uint32_t)swizzle};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return true;
  }
  if (!make_map(map, ptr, inner, outer, ld, box_inner, box_outer, swizzle)) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *map);
  return true;
}

// 4-D fp32 tensor map (no swizzle): the conv input batch as (x, y, image,
// channel) with element strides 1, width, img_stride, ch_stride -- both the
// image-major and the column-interleaved batch layouts; out-of-bounds
// elements read 0 (the conv's padding).  Cached per host thread.
bool cached_map4(CUtensorMap *map, const float *ptr, uint64_t width, uint64_t height,
                 uint64_t images, uint64_t channels, uint64_t img_stride, uint64_t ch_stride,
                 uint32_t box_x, uint32_t box_y, uint32_t box_c) {
  struct Key {
    const void *ptr;
    uint64_t v[8];
    bool operator==(const Key &o) const {
      if (ptr != o.ptr) return false;
      for (int i = 0; i < 8; ++i)
        if (v[i] != o.v[i]) return false;
      return true;
    }
  };
  struct Hash {
    size_t operator()(const Key &k) const {
      uint64_t h = reinterpret_cast<uint64_t>(k.ptr) * 0x9E3779B97F4A7C15ull;
      for (uint64_t x : k.v) h ^= x + 0x9E3779B9 + (h << 6) + (h >> 2);
      return (size_t)h;
    }
  };
  static thread_local std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key key{ptr, {width, height, images, channels, img_stride, ch_stride,
                      ((uint64_t)box_x << 32) | box_y, box_c}};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return true;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {width, height, images, channels};
  cuuint64_t strides[3] = {width * 4, img_stride * 4, ch_stride * 4};
  cuuint32_t box[4] = {box_x, box_y, 1, box_c};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if (fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(ptr), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 1024) cache.clear();
  cache.emplace(key, *map);
  return true;
}

// split-K scratch, one per (device, stream) so concurrent streams never share it.
// Grow-only, and a replaced buffer is RETIRED, never freed: a CUDA graph
// captured earlier on this stream keeps the old pointer (executor schedule
// cache), and replaying it after a larger uncaptured launch moved the
// workspace must still find valid memory.  Stream order keeps the old and
// new buffers' users apart.  The retired buffers are a few MB each.
std::mutex g_scratch_mu;
std::unordered_map<uint64_t, std::pair<float *, size_t>> g_scratch;
std::vector<float *> g_scratch_retired;

int scratch_for(cudaStream_t s, size_t floats, float **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t key = (reinterpret_cast<uint64_t>(s) << 8) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  auto &sc = g_scratch[key];
  if (sc.second < floats) {
    if (sc.first) g_scratch_retired.push_back(sc.first);
    sc.first = nullptr;
    sc.second = 0;
    if (int rc = check_cuda(cudaMalloc(&sc.first, floats * sizeof(float)), "gemm_tc: workspace"))
      return rc;
    sc.second = floats;
  }
  *out = sc.first;
  return ACCT_OK;
}

// stream-K tile counters: one int per (tile, CTA of the pair), zero between
// launches (the segment completing a tile resets it), per (device, stream)
// like the workspace
std::unordered_map<uint64_t, std::pair<int *, size_t>> g_sk_flags;

int sk_flags_for(cudaStream_t s, size_t n, int **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t key = (reinterpret_cast<uint64_t>(s) << 8) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  auto &f = g_sk_flags[key];
  if (f.second < n) {
    if (f.first) g_scratch_retired.push_back(reinterpret_cast<float *>(f.first));
    f.first = nullptr;
    f.second = 0;
    if (int rc = check_cuda(cudaMalloc(&f.first, n * sizeof(int)), "gemm_tc2: stream-K flags"))
      return rc;
    if (int rc = check_cuda(cudaMemset(f.first, 0, n * sizeof(int)), "gemm_tc2: stream-K flags"))
      return rc;
    f.second = n;
  }
  *out = f.first;
  return ACCT_OK;
}

// the row-band conv's weight image, per (device, stream), grow-only and
// retired like the workspace (a captured graph keeps its pointer)
std::unordered_map<uint64_t, std::pair<float *, size_t>> g_conv_w;

int conv_weights_for(cudaStream_t s, size_t floats, float **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t key = (reinterpret_cast<uint64_t>(s) << 8) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  auto &w = g_conv_w[key];
  if (w.second < floats) {
    if (w.first) g_scratch_retired.push_back(w.first);
    w.first = nullptr;
    w.second = 0;
    if (int rc = check_cuda(cudaMalloc(&w.first, floats * sizeof(float)), "conv_tc rows: weights"))
      return rc;
    w.second = floats;
  }
  *out = w.first;
  return ACCT_OK;
}

// co-resident 2-CTA clusters of a kernel on this device (cached per kernel)
template <typename Kern>
int sk_pairs(Kern kernel, int smem) {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (sm_count() / 2));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int cap = sm_count() / 2;
  if (n > cap) n = cap;
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

template <int TN, bool SWAP, int BK>
int set_smem_attr() {
  // the attribute is per device context
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    if (int rc = check_cuda(cudaFuncSetAttribute(tc_gemm_kernel<TN, SWAP, BK>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 Pick<TN, SWAP, BK>::G::SMEM_BYTES),
                            "gemm_tc: smem attribute"))
      return rc;
    done[dev] = true;
  }
  return ACCT_OK;
}

// fill the machine: split K until tiles x splits covers the SMs, keeping
// >= 2 k-blocks per split so the pipeline has something to overlap
int min_splits() {  // experiment knob (ACCT_TC_MINSPLIT): accuracy vs K-chunking
  static const int v = [] {
    const char *e = getenv("ACCT_TC_MINSPLIT");
    return e ? atoi(e) : 1;
  }();
  return v;
}

void plan_splits(int tiles, int total_kb, int sms, int *splits_out, int *kb_per_out) {
  int splits = 1;
  if (tiles < sms) {
    splits = sms / tiles;
    if (splits > total_kb / 2) splits = total_kb / 2;
    if (splits < 1) splits = 1;
  }
  if (splits < min_splits()) splits = min_splits() < total_kb ? min_splits() : total_kb;
  static const int max_kb = [] {  // ACCT_TC_MAXKB: cap k-blocks per split (accuracy knob)
    const char *e = getenv("ACCT_TC_MAXKB");
    return e ? atoi(e) : 0;
  }();
  if (max_kb > 0 && (total_kb + splits - 1) / splits > max_kb) splits = (total_kb + max_kb - 1) / max_kb;
  const int kb_per = (total_kb + splits - 1) / splits;
  *splits_out = (total_kb + kb_per - 1) / kb_per;
  *kb_per_out = kb_per;
}

// critical-path estimate of a normal-orientation launch with TN-wide tiles:
// waves x k-blocks per unit x TN (MMA time per k-block grows with TN)
int64_t tile_cost(int M, int N, int K, int TN, int BK, int sms) {
  const int tiles = ((M + 127) / 128) * ((N + TN - 1) / TN);
  int splits, kb_per;
  plan_splits(tiles, (K + BK - 1) / BK, sms, &splits, &kb_per);
  const int64_t waves = ((int64_t)tiles * splits + sms - 1) / sms;
  return waves * kb_per * BK * TN;
}

template <int TN, bool SWAP, int BK>
int launch_tc(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
              int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
              cudaStream_t s) {
  using G = typename Pick<TN, SWAP, BK>::G;
  CUtensorMap ta, tb;
  const uint32_t a_rows = SWAP ? TN : 128;  // weights: K-major box (BK k) x rows
  const CUtensorMapSwizzle kswz = BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!cached_map(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BK, a_rows, kswz) ||
      !cached_map(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, 32, BK,
                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return fail(ACCT_ENOTSUP, "gemm_tc: cuTensorMapEncodeTiled failed");
  const int tile_n = SWAP ? 128 : TN, tile_m = SWAP ? TN : 128;
  const int nt = (N + tile_n - 1) / tile_n, mt = (M + tile_m - 1) / tile_m, tiles = mt * nt;
  const int total_kb = (K + BK - 1) / BK;
  const int sms = sm_count();
  int splits, kb_per;
  plan_splits(tiles, total_kb, sms, &splits, &kb_per);
  const int units = tiles * splits;

  float *ws = nullptr;
  const int64_t ws_ld = (int64_t)nt * tile_n, rows = (int64_t)mt * tile_m;
  if (splits > 1) {
    if (int rc = scratch_for(s, (size_t)splits * rows * ws_ld, &ws)) return rc;
  }
  if (int rc = set_smem_attr<TN, SWAP, BK>()) return rc;
  const int grid = units < sms ? units : sms;
  launch(tc_gemm_kernel<TN, SWAP, BK>, dim3(grid), dim3(THREADS), G::SMEM_BYTES, s, ta, tb, M, N,
         K, nt, mt, splits, kb_per, g_write_hi | (prefetch_distance() << 8), alpha, beta, C, ldc, bias, act, ws, ws_ld,
         rows * ws_ld);
  if (int rc = note_launch("gemm_tc")) return rc;
  if (splits > 1) {
    const int64_t work = (int64_t)M * ((N + 3) / 4);
    launch(splitk_reduce_kernel, dim3(grid_for(work, 256)), dim3(256), 0, s, (const float *)ws, ws_ld,
           rows * ws_ld, splits, M, N, alpha, beta, C, ldc, bias, act);
    if (int rc = note_launch("gemm_tc_splitk_reduce")) return rc;
  }
  return ACCT_OK;
}

// 3-D fp32 tensor map of a conv input for the implicit-B gemm: (pixels of
// one plane, images, channels), box SEG pixels x 1 image x SLAB_CH channels;
// out-of-bounds pixels / channels read 0
bool make_input_map(CUtensorMap *map, const ImB &ib, int batch, uint32_t seg, uint32_t nch) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const uint64_t hw = (uint64_t)ib.H * ib.W;
  const uint64_t img_stride = batch > 1 ? (uint64_t)ib.act_img : ((hw + 3) & ~3ull);
  cuuint64_t dims[3] = {hw, (cuuint64_t)batch, (cuuint64_t)ib.cin};
  cuuint64_t strides[2] = {img_stride * 4, (uint64_t)ib.act_ld * 4};
  cuuint32_t box[3] = {seg, 1, nch};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(ib.act), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TN, int NACC, int BK, bool SWAP = false, bool DUAL = false, bool LOA = false,
          int PK = 0, bool IMB = false>
int launch_tc2(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
               int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
               cudaStream_t s, const ImB *imb = nullptr, const CUtensorMap *bmap = nullptr) {
  using G = Cfg2<TN, NACC, BK, SWAP, DUAL, LOA, PK, IMB>;
  CUtensorMap ta, tb;
  // weights: K-major box of BK x (128 rows, or TN/2 rows per CTA when swapped)
  if (!cached_map(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BK, SWAP ? TN / 2 : 128,
                  BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) ||
      (!IMB && !cached_map(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, 32, BK,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)))
    return fail(ACCT_ENOTSUP, "gemm_tc2: cuTensorMapEncodeTiled failed");
#ifdef ACCT_DBG_TBTA
  if (IMB) tb = ta;
#else
  if (IMB) tb = *bmap;  // the conv input: the split warps gather B from its slabs
#endif
  const ImB ib = imb ? *imb : ImB{};
  const int tile_n = SWAP ? 256 : TN, tile_m = SWAP ? TN : 256;
  const int nt = (N + tile_n - 1) / tile_n, mt = (M + tile_m - 1) / tile_m, tiles = mt * nt;
  const int total_kb = (K + BK - 1) / BK;
  const int pairs_avail = sm_count() / 2;
  // stream-K (chunked promotion only) when there are at least as many tiles
  // as CTA pairs: it removes the last wave's quantization.  With fewer tiles
  // split-K keeps the m-tiles of one column block at the same k at the same
  // time, so their shared B slices are L2 hits; a stream-K range per pair
  // puts them at unrelated k and re-reads B from HBM (yolov2-tiny L13,
  // 512 x 2749 x 9216: 128 vs 111 us; tools/sk_probe.py)
  const bool stream_k = PK > 0 && tiles >= pairs_avail;
  int splits = 1, kb_per = total_kb;
  if (!stream_k) plan_splits(tiles, total_kb, pairs_avail, &splits, &kb_per);
  const int units = tiles * splits;
  float *ws = nullptr;
  const int64_t ws_ld = (int64_t)nt * tile_n, rows = (int64_t)mt * tile_m;
  if (splits > 1) {
    if (int rc = scratch_for(s, (size_t)splits * rows * ws_ld, &ws)) return rc;
  }
  {
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      if (int rc = check_cuda(cudaFuncSetAttribute(tc2_gemm_kernel<TN, NACC, BK, SWAP, DUAL, LOA, PK, IMB>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   G::SMEM_BYTES),
                              "gemm_tc2: smem attribute"))
        return rc;
      done[dev] = true;
    }
  }
  int pairs = units < pairs_avail ? units : pairs_avail;
  int *flags = nullptr;
  if (stream_k) {
    // stream-K: every pair gets an equal share of the (tile, chunk) space;
    // the grid is the clusters that fit at once (one wave of pairs)
    const int cpt = (total_kb + PK - 1) / PK;
    const int64_t tot_ch = (int64_t)tiles * cpt;
    pairs = sk_pairs(tc2_gemm_kernel<TN, NACC, BK, SWAP, DUAL, LOA, PK, IMB>, G::SMEM_BYTES);
    if (pairs < 1) return fail(ACCT_ENOTSUP, "gemm_tc2 stream-K: no co-resident CTA pairs");
    if (tot_ch < pairs) pairs = (int)tot_ch;
    if (int rc = scratch_for(s, (size_t)4 * pairs * 128 * TN, &ws)) return rc;
    if (int rc = sk_flags_for(s, 2 * (size_t)tiles, &flags)) return rc;
  }
  launch(tc2_gemm_kernel<TN, NACC, BK, SWAP, DUAL, LOA, PK, IMB>, dim3(2 * pairs), dim3(THREADS),
         G::SMEM_BYTES, s, ta, tb, M, N, K, nt, mt, splits, kb_per, g_write_hi, alpha, beta, C, ldc,
         bias, act, ws, ws_ld, rows * ws_ld, flags, ib);
  if (int rc = note_launch("gemm_tc2")) return rc;
  if (splits > 1) {
    const int64_t work = (int64_t)M * ((N + 3) / 4);
    launch(splitk_reduce_kernel, dim3(grid_for(work, 256)), dim3(256), 0, s, (const float *)ws, ws_ld,
           rows * ws_ld, splits, M, N, alpha, beta, C, ldc, bias, act);
    if (int rc = note_launch("gemm_tc_splitk_reduce")) return rc;
  }
  return ACCT_OK;
}

// critical path of a CTA-pair launch (each SM: 128 rows x TN per k-block)
int64_t tile_cost2(int M, int N, int K, int TN, int BK, int pairs) {
  const int tiles = ((M + 255) / 256) * ((N + TN - 1) / TN);
  int splits, kb_per;
  plan_splits(tiles, (K + BK - 1) / BK, pairs, &splits, &kb_per);
  const int64_t waves = ((int64_t)tiles * splits + pairs - 1) / pairs;
  return waves * kb_per * BK * TN;
}

}  // namespace

int gemm_tc(int M, int N, int K, float alpha, const float *A, int64_t lda, const float *B,
            int64_t ldb, float beta, float *C, int64_t ldc, const float *bias, int act,
            cudaStream_t s) {
  // TMA needs 16-B aligned bases and row pitches
  if (M < 1 || N < 1 || K < 1 || (lda % 4) || (ldb % 4) ||
      (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
    return ACCT_ENOTSUP;
  if (M <= 16) return launch_tc<16, true, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  // swap tiles, single SM by default; 12 forces the CTA-pair swap tile.  The
  // pair does not pay here: a 128 x 32 x 8 MMA issues in ~69 cycles and a
  // 256 x 32 x 8 pair MMA in ~82 (tools/tc_trace.py), both far above the 16
  // cycles of math, so narrow tiles stay MMA-issue bound either way.
  const int fswap = forced_tile();
  if (M <= 32)
    return fswap == 12 ? launch_tc2<32, 4, 32, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s)
                       : launch_tc<32, true, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (M <= 64)
    return fswap == 12 ? launch_tc2<64, 4, 32, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s)
                       : launch_tc<64, true, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  const int force = forced_tile();
  if (force == 1) return launch_tc<192, false, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 2) return launch_tc<128, false, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 3) return launch_tc<128, false, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 4) return launch_tc<256, false, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 5) return launch_tc2<192, 2, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 6) return launch_tc2<256, 1, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 7) return launch_tc2<128, 2, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 8) return launch_tc2<192, 1, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 9) return launch_tc2<192, 1, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 10) return launch_tc2<256, 1, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 13) return launch_tc2<192, 1, 16, false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 14) return launch_tc2<128, 1, 32, false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (force == 15) return launch_tc2<192, 1, 32, false, true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  // Candidates: one SM per 128 x 192 tile (operand A in TMEM), or a CTA pair
  // per 256 x {192, 256} tile (cta_group::2, BK = 32).  Pick the shortest
  // critical path -- waves x k-blocks per unit x TN after split-K -- with the
  // single-SM tile weighted by its measured shared-memory-bound efficiency
  // (743 vs ~590 cycles per 128x192x16 k-block, tools/tc_trace.py).
  const int sms = sm_count();
  const double c1 = 1.25 * (double)tile_cost(M, N, K, 192, 16, sms);
  // a pair tile spans 256 rows: weight its cost by the rows it computes vs
  // the 128-row tiles (M = 128 would waste half of every pair)
  const double waste = (double)((M + 255) / 256 * 256) / (double)((M + 127) / 128 * 128);
  const double c9 = waste * (double)tile_cost2(M, N, K, 192, 32, sms / 2);
  const double c10 = waste * (double)tile_cost2(M, N, K, 256, 32, sms / 2);
  // Long K: the tensor core's truncating FP32 accumulate compounds (3xTF32
  // relative error ~1e-5 at K = 4608, enough to pass 1e-4 through the 26
  // layers of yolov2-608: 1.46e-4 at 16 images with a second accumulator for
  // the small terms, "DUAL", force 16).  Above kDualK (768: every pair-tile
  // layer of the nets but the shortest) the pair tile promotes the
  // accumulator every 4 k-blocks into an FP32 register sum (PK = 4, only A lo
  // in TMEM): yolov2-608 5.5e-5, yolov2-tiny 1.6e-5 (was 3.7e-5), and 3%
  // faster than DUAL (its single accumulator stalled the MMAs at every unit
  // boundary).  Chunks of 2 / 1 k-blocks: 4.9e-5 / 4.6e-5 at 17% / 37% more
  // time -- the remaining error is elsewhere (tools/err_dist.py).
  constexpr int kDualK = 768;
  if (force == 17)  // the chunked-promotion pair tile whatever the cost model says (tests)
    return launch_tc2<192, 2, 32, false, false, true, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if ((c10 < c1 || c9 < c1) && K > kDualK) {
    if (force == 16)  // the previous default (DUAL, no promotion), for comparison
      return launch_tc2<192, 1, 32, false, true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);

    return launch_tc2<192, 2, 32, false, false, true, 4>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  }
  if (c10 < c9 && c10 < c1)
    return launch_tc2<256, 1, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  if (c9 < c1)
    return launch_tc2<192, 1, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
  return launch_tc<192, false, 16>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias, act, s);
}

// optional 2x2/2 maxpool of the conv output, fused into the epilogue
struct ConvPool {
  float *pool;
  int64_t ld_pool, pool_stride;
  int32_t *idx;
  int64_t ld_idx, idx_stride;
  int c_from;  // C stored for images >= c_from only (the pooled copies are dead)
};

// Implicit-im2col conv on tensor cores (tc_conv_kernel): M <= 64 filters,
// channels <= 64, any batch layout with 16-B aligned strides; ENOTSUP when
// the resident weights and the two slabs exceed shared memory.
template <int TN, int TW>
int launch_conv_tc(const float *im, int64_t ld_im, int64_t im_stride, int channels, int height,
                   int width, float *col, int64_t ld_col, int64_t col_stride, int M,
                   const float *A, int64_t lda, float beta, float *C, int64_t ldc,
                   int64_t c_stride, const float *bias, int act, int batch, int col_from,
                   const ConvPool &pl, cudaStream_t s) {
  using G = ConvCfg<TN, TW>;
  const int K = 9 * channels;
  const int nkb = (K + G::BK - 1) / G::BK;
  const size_t slab_bytes = ((size_t)channels * G::CS + 127) & ~size_t(127);
  // a deeper slab ring keeps several units' input windows in flight: the
  // first layers (K = 27) have one k-block per unit and are latency-bound
  const size_t fixed = 1024 + 2 * (size_t)nkb * G::W_TILE + 8 * (1 + 2 * kMaxSlabs +
                       2 * G::NP * G::S + 2 * G::NP * G::NACC) + 32 + 4 * 64 +
                       (pl.pool ? 4 * 8 * 8 * 33 : 0);
  if (fixed + 2 * slab_bytes > 227 * 1024) return ACCT_ENOTSUP;
  int nslab = (int)((227 * 1024 - fixed) / slab_bytes);
  if (nslab > kMaxSlabs) nslab = kMaxSlabs;
  const size_t smem = fixed + (size_t)nslab * slab_bytes;
  CUtensorMap tw, tx;
  if (!cached_map(&tw, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, G::BK, TN,
                  CU_TENSOR_MAP_SWIZZLE_128B) ||
      !cached_map4(&tx, im, (uint64_t)width, (uint64_t)height, (uint64_t)batch,
                   (uint64_t)channels, (uint64_t)(batch > 1 ? im_stride : ld_im), (uint64_t)ld_im,
                   G::TWP, G::SROWS, channels))
    return fail(ACCT_ENOTSUP, "conv_tc: cuTensorMapEncodeTiled failed");
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      for (auto k : {tc_conv_kernel<TN, TW, false>, tc_conv_kernel<TN, TW, true>})
        if (int rc = check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     227 * 1024),
                                "conv_tc: smem attribute"))
          return rc;
      done[dev] = true;
    }
  }
  const int tiles_x = (width + TW - 1) / TW, tiles_y = (height + G::TH - 1) / G::TH;
  const int64_t tpi = (int64_t)tiles_x * tiles_y;
  const int64_t units = tpi * batch;
  if (units >= (1 << 24)) return ACCT_ENOTSUP;  // acct_divmod
  const int sms = sm_count();
  const int grid = units < sms ? (int)units : sms;
  static const int dbg = [] {  // bit 64: clock64 trace (tools/conv_trace.py); the work-skipping
    const char *e = getenv("ACCT_CONV_DBG");  // bits 1-32 need the -DACCT_PROFILING build
    return e ? atoi(e) : 0;
  }();
  launch(beta != 0.0f ? tc_conv_kernel<TN, TW, true> : tc_conv_kernel<TN, TW, false>, dim3(grid),
         dim3(CONV_NARROW_THREADS), smem, s, tw, tx, M, channels,
         height, width, tiles_x, (int)tpi, (int)units, nkb, beta, C, ldc, c_stride, bias, act, col,
         ld_col, col_stride, col_from, pl.pool, pl.ld_pool, pl.pool_stride, pl.idx, pl.ld_idx,
         pl.idx_stride, pl.c_from, nslab, dbg);
  return note_launch("conv3x3 tc");
}

// wide layers: M a multiple of 128 (filter blocks), any channel count
template <int TW>
int launch_conv_wide(const float *im, int64_t ld_im, int64_t im_stride, int channels, int height,
                     int width, float *col, int64_t ld_col, int64_t col_stride, int M,
                     const float *A, int64_t lda, float beta, float *C, int64_t ldc,
                     int64_t c_stride, const float *bias, int act, int batch, int col_from,
                     const ConvPool &pl, cudaStream_t s) {
  using G = WideCfg<TW>;
  const int K = 9 * channels;
  const int nkb = (K + G::BK - 1) / G::BK;
  const size_t smem = 1024 + (size_t)G::S * G::STAGE + 8 * (3 * G::S + 2 * G::NACC) + 16 +
                      16 + 4 * 256 + (pl.pool ? 4 * 8 * 8 * 33 : 0);
  if (smem > 227 * 1024 || M % G::TN || M > 256) return ACCT_ENOTSUP;  // bias_s holds 256
  CUtensorMap tw, tx;
  if (!cached_map(&tw, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, G::BK, G::TN,
                  CU_TENSOR_MAP_SWIZZLE_128B) ||
      !cached_map4(&tx, im, (uint64_t)width, (uint64_t)height, (uint64_t)batch,
                   (uint64_t)channels, (uint64_t)(batch > 1 ? im_stride : ld_im), (uint64_t)ld_im,
                   G::TWP, G::SROWS, G::CH_PER_KB))
    return fail(ACCT_ENOTSUP, "conv_tc wide: cuTensorMapEncodeTiled failed");
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      for (auto k : {tc_conv_wide_kernel<TW, false>, tc_conv_wide_kernel<TW, true>})
        if (int rc = check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     227 * 1024),
                                "conv_tc wide: smem attribute"))
          return rc;
      done[dev] = true;
    }
  }
  const int tiles_x = (width + TW - 1) / TW, tiles_y = (height + G::TH - 1) / G::TH;
  const int64_t tpi = (int64_t)tiles_x * tiles_y;
  const int64_t units = tpi * batch * (M / G::TN);
  if (units >= (1 << 24)) return ACCT_ENOTSUP;  // acct_divmod
  const int sms = sm_count();
  const int grid = units < sms ? (int)units : sms;
  static const int dbg = [] {
    const char *e = getenv("ACCT_CONV_DBG");
    return e ? atoi(e) : 0;
  }();
  launch(beta != 0.0f ? tc_conv_wide_kernel<TW, true> : tc_conv_wide_kernel<TW, false>, dim3(grid),
         dim3(CONV_TC_THREADS), smem, s, tw, tx, M, channels,
         height, width, tiles_x, (int)tpi, (int)units, nkb, beta, C, ldc, c_stride, bias, act, col,
         ld_col, col_stride, col_from, pl.pool, pl.ld_pool, pl.pool_stride, pl.idx, pl.ld_idx,
         pl.idx_stride, pl.c_from, batch, dbg);
  return note_launch("conv3x3 tc wide");
}

// row-band conv (tc_conv_rows_kernel): M <= 32 filters (for 33..64 the
// im2col-operand kernel measured faster: the shared-memory operand reads of
// N = 64 MMAs bound this design, tools/conv_rows_probe.py), channels a
// multiple of 8 whose resident [W hi | W lo] leave room for two staging
// steps; col of images >= col_from written by the staging warps.
// ENOTSUP for other shapes (the caller falls back to tc_conv_kernel).
std::atomic<int> g_conv_rows{0};
int conv_dbg() {  // ACCT_CONV_DBG work-skipping bits: the -DACCT_PROFILING build only
  static const int dbg = [] {
    const char *e = getenv("ACCT_CONV_DBG");
    return e ? atoi(e) : 0;
  }();
  return dbg;
}

template <int TN>
int launch_conv_rows(const float *im, int64_t ld_im, int64_t im_stride, int channels, int height,
                     int width, float *col, int64_t ld_col, int64_t col_stride, int M,
                     const float *A, int64_t lda, float beta, float *C, int64_t ldc,
                     int64_t c_stride, const float *bias, int act, int batch, int col_from,
                     const ConvPool &pl, cudaStream_t s) {
  using G = RowsCfg<TN>;
  if (!g_conv_rows.load(std::memory_order_relaxed) || channels % 8 || M > TN) return ACCT_ENOTSUP;
  const int nstrips = (width + 127) / 128;
  int swd = (width + nstrips - 1) / nstrips;
  swd += swd & 1;  // even: pooling windows never straddle strips
  const int sp = swd + 2;
  const int pairs = (height + 1) / 2;
  const int64_t units = (int64_t)batch * nstrips * pairs;
  if (units > INT32_MAX) return ACCT_ENOTSUP;
  const size_t stage_bytes = 256 * (size_t)sp;
  const size_t w_bytes = (size_t)9 * channels * 2 * TN * 4;
  // (the MMA rows past wdt read up to 130 - sp positions beyond the last
  // stage: into the weights, never outside the block; those rows are dropped)
  const size_t fixed = 1024 + w_bytes + 4 * TN + 8 * (2 * G::MAXS + 2 * G::NACC + 1) + 16;
  if (fixed + 2 * stage_bytes > 227 * 1024) return ACCT_ENOTSUP;
  int nstage = (int)((227 * 1024 - fixed) / stage_bytes);
  if (nstage > G::MAXS) nstage = G::MAXS;
  const size_t smem = fixed + (size_t)nstage * stage_bytes;
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      if (int rc = check_cuda(cudaFuncSetAttribute(tc_conv_rows_kernel<TN>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   227 * 1024),
                              "conv_tc rows: smem attribute"))
        return rc;
      done[dev] = true;
    }
  }
  float *wimg = nullptr;
  if (int rc = conv_weights_for(s, w_bytes / 4, &wimg)) return rc;
  {
    const int items = 9 * (channels / 4) * TN;
    launch(rows_weights_kernel<TN>, dim3((items + 255) / 256), dim3(256), 0, s, A, lda, M,
           channels, reinterpret_cast<float4 *>(wimg));
    if (int rc = note_launch("conv3x3 tc rows weights")) return rc;
  }
  const int sms = sm_count();
  const int grid = units < sms ? (int)units : sms;
  launch(tc_conv_rows_kernel<TN>, dim3(grid), dim3(ROWS_THREADS), smem, s, im, ld_im,
         batch > 1 ? im_stride : (int64_t)0, channels, height, width,
         reinterpret_cast<const float4 *>(wimg), M, col_from < batch ? col : nullptr, ld_col,
         col_stride, col_from, nstrips, swd, sp,
         pairs, (int)units, nstage, beta, C, ldc, c_stride, bias, act, pl.pool, pl.ld_pool,
         pl.pool_stride, pl.idx, pl.ld_idx, pl.idx_stride, pl.c_from, conv_dbg());
  return note_launch("conv3x3 tc rows");
}

template <int TN>
int conv_tc(const float *im, int64_t ld_im, int64_t im_stride, int channels, int height,
            int width, float *col, int64_t ld_col, int64_t col_stride, int M, const float *A,
            int64_t lda, float beta, float *C, int64_t ldc, int64_t c_stride, const float *bias,
            int act, int batch, int col_from, const ConvPool &pl, cudaStream_t s) {
  if constexpr (TN == 32) {  // the row-band kernel (opt-in) takes M <= 32 only
    const int rc = launch_conv_rows<TN>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                                        col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act,
                                        batch, col_from, pl, s);
    if (rc != ACCT_ENOTSUP) return rc;
  }
  // 16-wide pixel blocks unless the width is a multiple of 8 but not of 16;
  // the other width when those slabs do not fit next to the pooling scratch
  const bool eight = width % 16 != 0 && width % 8 == 0;
  int rc = eight ? launch_conv_tc<TN, 8>(im, ld_im, im_stride, channels, height, width, col,
                                         ld_col, col_stride, M, A, lda, beta, C, ldc, c_stride,
                                         bias, act, batch, col_from, pl, s)
                 : launch_conv_tc<TN, 16>(im, ld_im, im_stride, channels, height, width, col,
                                          ld_col, col_stride, M, A, lda, beta, C, ldc, c_stride,
                                          bias, act, batch, col_from, pl, s);
  if (rc == ACCT_ENOTSUP && eight)
    rc = launch_conv_tc<TN, 16>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                                col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act, batch,
                                col_from, pl, s);
  return rc;
}

}  // namespace acct

extern "C" void acct_tc_set_write_hi(int on) { acct::g_write_hi = on; }

// co-resident CTA pairs of the stream-K gemm on the current device (diagnostics)
extern "C" int acct_tc_stream_k_pairs(void) {
  using G = acct::Cfg2<192, 2, 32, false, false, true, 4>;
  return acct::sk_pairs(acct::tc2_gemm_kernel<192, 2, 32, false, false, true, 4, false>,
                        G::SMEM_BYTES);
}

// 1: narrow convs with M <= 32 on the row-band kernel instead of the
// im2col-operand kernel (default 0: measured no faster in the nets)
// -- tests / A-B measurements only
extern "C" void acct_tc_set_conv_rows(int on) { acct::g_conv_rows.store(on ? 1 : 0); }

extern "C" void acct_tc_set_tile(int tile) { acct::g_force_tile.store(tile < 0 ? 0 : tile); }

extern "C" int acct_tc_trace(long long *out) {
  return acct::check_cuda(cudaMemcpyFromSymbol(out, acct::g_trace, sizeof(acct::g_trace)),
                          "tc trace");
}

// C = A . im2col(im) + beta C (+ bias, act) for 3x3/1/1 convolutions with
// M <= 64 filters on tcgen05 (3xTF32, the swap tile's arithmetic), col stored
// for images >= col_from of the batch; ENOTSUP for shapes it does not take
extern "C" int acct_conv3x3_tc_f32(const float *im, int64_t ld_im, int64_t im_stride,
                                   int channels, int height, int width, float *col,
                                   int64_t ld_col, int64_t col_stride, int M, const float *A,
                                   int64_t lda, float beta, float *C, int64_t ldc,
                                   int64_t c_stride, const float *bias, int act, int batch,
                                   int col_from, float *pool, int64_t ld_pool,
                                   int64_t pool_stride, int32_t *idx, int64_t ld_idx,
                                   int64_t idx_stride, int c_from, acct_stream_t stream) {
  using namespace acct;
  if (channels < 1 || channels > 1024 || M < 1 || (M > 64 && M % 128) || height < 1 ||
      width < 1 || batch < 1 || col_from < 0 || c_from < 0 || (int64_t)height * width > (1 << 28) ||
      ld_im < (int64_t)height * width || ld_col < (int64_t)height * width ||
      ldc < (int64_t)height * width || (batch > 1 && (im_stride < 1 || (im_stride & 3))))
    return fail(ACCT_ENOTSUP, "conv3x3 tc: shape not supported");
  if ((reinterpret_cast<uintptr_t>(im) | reinterpret_cast<uintptr_t>(A)) & 15 ||
      (ld_im | lda) & 3)
    return fail(ACCT_ENOTSUP, "conv3x3 tc: needs 16-B aligned operands");
  if (pool && (!idx || (height | width) & 1 ||
               ld_pool < (int64_t)(height / 2) * (width / 2) ||
               ld_idx < (int64_t)(height / 2) * (width / 2)))
    return fail(ACCT_ENOTSUP, "conv3x3 tc: fused maxpool needs even planes");
  if (!pool) c_from = 0;
  const ConvPool pl{pool, ld_pool, pool_stride, idx, ld_idx, idx_stride, c_from};
  cudaStream_t s = as_stream(stream);
  int rc;
  if (M > 64) {
    const bool eight = width % 16 != 0 && width % 8 == 0;
    rc = eight ? launch_conv_wide<8>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                                     col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act,
                                     batch, col_from, pl, s)
               : launch_conv_wide<16>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                                      col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act,
                                      batch, col_from, pl, s);
  } else if (channels > 64) {
    rc = ACCT_ENOTSUP;
  } else {
    rc = M <= 32 ? conv_tc<32>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                               col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act, batch,
                               col_from, pl, s)
                 : conv_tc<64>(im, ld_im, im_stride, channels, height, width, col, ld_col,
                               col_stride, M, A, lda, beta, C, ldc, c_stride, bias, act, batch,
                               col_from, pl, s);
  }
  if (rc == ACCT_ENOTSUP)
    return fail(ACCT_ENOTSUP, "conv3x3 tc: weights + slabs exceed shared memory");
  return rc;
}

// C = A . im2col(im) + beta C (+ bias, act) for 3x3/1/1 convolutions with
// many filters and a long K (M >= 256, 9 channels > 768): the CTA-pair
// chunked-promotion gemm with operand B gathered from the input planes
// (implicit im2col, ImB) -- bit-identical to acct_im2col_batched_f32 + the
// same gemm; col stored for images >= col_from.  C and col must be
// column-interleaved with one image pitch (c_stride == col_stride); the input
// may use any image stride.  ENOTSUP for other shapes and for a fused pool.
extern "C" int acct_conv3x3_gemm_tc_f32(const float *im, int64_t ld_im, int64_t im_stride,
                                        int channels, int height, int width, float *col,
                                        int64_t ld_col, int64_t col_stride, int M,
                                        const float *A, int64_t lda, float beta, float *C,
                                        int64_t ldc, int64_t c_stride, const float *bias,
                                        int act, int batch, int col_from, float *pool,
                                        int64_t ld_pool, int64_t pool_stride, int32_t *idx,
                                        int64_t ld_idx, int64_t idx_stride, int c_from,
                                        acct_stream_t stream) {
  using namespace acct;
  (void)ld_pool, (void)pool_stride, (void)idx, (void)ld_idx, (void)idx_stride, (void)c_from;
  const int64_t HW = (int64_t)height * width;
  const int K = 9 * channels;
  if (pool || M < 256 || K <= 768 || channels < 1 || height < 1 || width < 1 || batch < 1 ||
      col_from < 0 || HW > (1 << 24) || ldc < HW || ld_col < HW ||
      (batch > 1 && (c_stride < HW || col_stride != c_stride)) || (lda & 3) ||
      (reinterpret_cast<uintptr_t>(A) & 15))
    return fail(ACCT_ENOTSUP, "conv3x3 implicit gemm: shape not supported");
  const int64_t n_img = batch > 1 ? c_stride : 0;
  const int64_t N = (int64_t)(batch - 1) * n_img + HW;
  if (N > INT32_MAX) return fail(ACCT_ENOTSUP, "conv3x3 implicit gemm: too many columns");
  using G = Cfg2<192, 2, 32, false, false, true, 4, true>;
  // a CTA's half tile must touch <= 2 images and its pixels +- one row must
  // fit one slab segment
  if ((batch > 1 && n_img < G::HALF) || G::HALF + 2 * width + 5 > G::SEG ||
      (batch > 1 && (im_stride & 3)) || (ld_im & 3) || (reinterpret_cast<uintptr_t>(im) & 15))
    return fail(ACCT_ENOTSUP, "conv3x3 implicit gemm: plane layout not supported");
  ImB ib;
  ib.act = im;
  ib.act_ld = ld_im;
  ib.act_img = batch > 1 ? im_stride : 0;
  ib.img = n_img;
  ib.cin = channels;
  ib.H = height;
  ib.W = width;
  ib.col = col_from < batch ? col : nullptr;
  ib.col_ld = ld_col;
  ib.col_n0 = (int64_t)col_from * n_img;
  CUtensorMap bmap;
  if (!make_input_map(&bmap, ib, batch, G::SEG, G::SLAB_CH))
    return fail(ACCT_ENOTSUP, "conv3x3 implicit gemm: input tensor map");
  return launch_tc2<192, 2, 32, false, false, true, 4, true>(
      M, (int)N, K, 1.0f, A, lda, nullptr, 0, beta, C, ldc, bias, act, as_stream(stream), &ib,
      &bmap);
}
