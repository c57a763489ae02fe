// softmin_hd.cu — K1h: the softmin for high feature dimension (D <= 64; the
// D = 60 fibre features of config 4) with the <x, y> term
// on the 5th-generation tensor cores.
//
//   f_i = -lambda eps log sum_j w_j exp((h_j + est_i/lambda... ) ), written as
//   E_ij = c_j + r_i + <x_i, y_j> / (eps ln2)            (log2 units)
//   c_j  = log2 w_j + (h_j - |y_j|^2 / 2) / (eps ln2),   r_i = est_i/(lambda eps ln2) - |x_i|^2/(2 eps ln2)
//
// Precision: a single TF32/F16 product has ~2^-11 relative error, i.e. an
// error of ~0.5 in E at blur 0.03 — far outside the 1e-3 eps tolerance.  Each
// coordinate (centred, x 2^6) is split x = hi + lo into two float16s and the
// MMA computes hi.hi + hi.lo + lo.hi (relative error ~2^-22): three K = 64
// products into one accumulator.  Every atom is packed once as [hi | lo]
// (2 x 16 KB per 128 atoms) and serves as A (rows) or B (columns).
//
// Kernel (one CTA per work item = 256 rows x a run of 128-column blocks):
//   warp 0      producer: cp.async.bulk (TMA) of the pre-swizzled operands
//               (A once, B per stage, kHdStages stages) and of the block's
//               128 column constants c_j (hd_colconst) into a 2-slot ring
//   warp 1      TMEM owner + MMA issuer: per column block, 2 M-halves x 3
//               products x 4 K-steps of tcgen05.mma.kind::f16 (M=128, N=128,
//               K=16) into a double-buffered 2 x 256-column fp32 accumulator
//   warps 2-17  epilogue, four warpgroups = 2 M-halves x 2 column halves;
//               one TMEM lane = one row per thread: tcgen05.ld 32x32b.x32,
//               E = k2 v + (c_j + r_i) on the packed FMA pipe, MUFU ex2,
//               running row sum; arrive on the TMEM-empty barrier
// Operands are K-major, 128-byte swizzled (SWIZZLE_128B, 1024-byte atoms):
// 16-byte chunk q of row r sits at r*128 + ((q ^ (r & 7)) * 16).
#include <cuda_fp16.h>

#include "prims.cuh"

namespace msot_dev {

constexpr int kHdK = 64;                 // f16 per 128-byte row (one swizzle atom)
constexpr int kHdParts = 2;              // [hi | lo]
constexpr int kHdBlockRows = 128;
constexpr int kHdBlockBytes = kHdBlockRows * 128;            // 16 KB
constexpr int kHdPackBytes = kHdParts * kHdBlockBytes;       // 32 KB per 128 atoms
constexpr int kHdEpiWarps = 16;
constexpr int kHdThreads = 64 + 32 * kHdEpiWarps;  // producer, MMA, 16 epilogue warps
constexpr float kHdScale = 64.f;         // coordinate scale before the f16 split

// Shared memory plan.  kSym (evaluate-once) adds a 4 KB per-warp transpose
// area and the cross-warp column accumulators, and keeps 2 B stages.
template <bool kSym>
struct HdSmem {
  static constexpr int kStages = kSym ? 2 : 3;
  static constexpr int kRing = kSym ? 256 : 128;  // floats per ring slot: c_j (+ column factors)
  static constexpr size_t kA = 0;
  static constexpr size_t kB = kA + 2 * kHdPackBytes;
  static constexpr size_t kStage = kB + kStages * kHdPackBytes;            // [16 warps][32][32] f32
  static constexpr size_t kColAcc = kStage + (kSym ? kHdEpiWarps * 4096 : 0);  // [2 buf][4 cq][4 q][32]
  static constexpr size_t kRingOff = kColAcc + (kSym ? 2 * 4 * 4 * 32 * 4 : 0);
  static constexpr size_t kRowAcc = kRingOff + 2 * kRing * 4;              // [4 cq][256]
  static constexpr size_t kBars = kRowAcc + 4 * kTileRows * 4;
  static constexpr size_t kTotal = kBars + 256 + 1024;                    // barriers, alignment
};
static_assert(HdSmem<true>::kTotal <= 227 * 1024, "shared memory");
static_assert(HdSmem<false>::kTotal <= 227 * 1024, "shared memory");

// ---------------------------------------------------------------- packing --
// One thread per (atom, 16-byte chunk): writes the chunk's 8 f16 of the hi
// and the lo part.  (`role` is kept for the call sites: A and B share the
// layout.)
__global__ void hd_pack_kernel(const double* x, int64_t n, int64_t npad, int d,
                               const double* center, int role, uint8_t* pack, float* sq,
                               float* xf) {
  (void)role;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= npad * 8) return;
  const int64_t i = g >> 3;
  const int q = static_cast<int>(g & 7);
  __half hi[8], lo[8];
  float part = 0.f;
  for (int e = 0; e < 8; ++e) {
    const int k = q * 8 + e;
    float v = 0.f;
    if (i < n && k < d) v = static_cast<float>(x[i * d + k] - center[k]);
    if (xf) xf[i * kHdK + k] = v;  // padded rows/dims are zero
    part = fmaf(v, v, part);
    const float vs = v * kHdScale;
    hi[e] = __float2half_rn(vs);
    lo[e] = __float2half_rn(vs - __half2float(hi[e]));
  }
  // |x|^2 from the float coordinates: reduce the 8 chunk partials (lanes 8i..8i+7)
  for (int o = 4; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (q == 0 && i < n && sq) sq[i] = part;
  const int64_t blk = i / kHdBlockRows;
  const int r = static_cast<int>(i % kHdBlockRows);
  const int off = r * 128 + ((q ^ (r & 7)) * 16);
  uint8_t* base = pack + blk * kHdPackBytes;
  *reinterpret_cast<uint4*>(base + off) = *reinterpret_cast<const uint4*>(hi);
  *reinterpret_cast<uint4*>(base + kHdBlockBytes + off) = *reinterpret_cast<const uint4*>(lo);
}

// Rows are padded to whole 256-row tiles (two A blocks per CTA), columns to
// whole 128-column blocks.
int64_t hd_padded(int64_t n) { return (n + kTileRows - 1) / kTileRows * kTileRows; }

cudaError_t hd_pack(const double* x, int64_t n, int d, const double* center, int role,
                    uint8_t* pack, float* sq, float* xf, cudaStream_t st) {
  const int64_t npad = hd_padded(n);
  const int64_t threads = npad * 8;
  ++g_launches;
  hd_pack_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      x, n, npad, d, center, role, pack, sq, xf);
  return cudaGetLastError();
}

size_t hd_pack_bytes(int64_t n) {
  return static_cast<size_t>(hd_padded(n) / kHdBlockRows) * kHdPackBytes;
}

// ----------------------------------------------------------- PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// K-major, SWIZZLE_128B UMMA shared-memory descriptor (SM100 version 1):
// start >> 4, LBO = 1 (unused for swizzled K-major), SBO = 1024 B >> 4.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}

// instruction descriptor: F16 x F16 -> F32, K-major A and B, M = 128, N = 128
constexpr uint32_t kHdIdesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---------------------------------------------------------------- kernel --
// kSym: evaluate-once (softmin_sym.cu's scheme on the dense high-D problems):
// every exponential also feeds its column.  Per 32 columns a warp stages its
// 32 x 32 block through shared memory (16-byte chunks XOR-swizzled by row),
// each lane sums 8 rows x 4 columns, two shuffle levels finish the warp's
// column sums, and after the block the 8 warps of a column half combine in
// a fixed order into colpart[tile slot + position] (column factor applied).
template <bool kSym>
__global__ void __launch_bounds__(kHdThreads, 1)
softmin_hd_kernel(const __grid_constant__ Group G) {
  using L = HdSmem<kSym>;
  extern __shared__ __align__(1024) uint8_t hd_smem_raw[];
  // align to 1024 B by offsetting the shared array itself, so the compiler
  // keeps every derived pointer in the shared window (LDS/STS, not generic)
  uint8_t* smem = hd_smem_raw + ((1024u - (smem_u32(hd_smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem + L::kA;
  uint8_t* sB = smem + L::kB;
  float* stage_all = reinterpret_cast<float*>(smem + L::kStage);
  float* colacc = reinterpret_cast<float*>(smem + L::kColAcc);
  float* cring = reinterpret_cast<float*>(smem + L::kRingOff);
  float* rowacc = reinterpret_cast<float*>(smem + L::kRowAcc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);
  // bars: 0 fullA | fullB[S] | emptyB[S] | tmemFull[2] | tmemEmpty[2] | cFull[2] | colFull[2][4]
  uint64_t* fullB = bars + 1;
  uint64_t* emptyB = fullB + L::kStages;
  uint64_t* tmemFull = emptyB + L::kStages;
  uint64_t* tmemEmpty = tmemFull + 2;
  uint64_t* cFull = tmemEmpty + 2;
  uint64_t* colFull = cFull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(colFull + 8);
  int32_t* ring_blk = reinterpret_cast<int32_t*>(tmem_slot + 1);  // [2] column block per ring slot

  const int it = blockIdx.x;
  if (it >= G.n_items) return;
  const int4 item = G.items[it];
  const Problem& P = G.P[item.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row_base = P.tile_start[item.y];
  // position blocks of this item: the 128-position blocks of the tile's
  // concatenated column ranges whose first position lies in [z, w).  Every
  // range starts and ends on a 128-column block (dense lists, padded K-means
  // clusters), so position block b maps to one whole column block.
  const int pb0 = (item.z + kHdBlockRows - 1) / kHdBlockRows;
  const int pb1 = (item.w + kHdBlockRows - 1) / kHdBlockRows;
  const int nblk = pb1 - pb0;

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(smem_u32(&fullB[s]), 1);
      mbar_init(smem_u32(&emptyB[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tmemFull[b]), 1);
      mbar_init(smem_u32(&tmemEmpty[b]), kHdEpiWarps);
      mbar_init(smem_u32(&cFull[b]), 1);
      for (int k = 0; k < 4; ++k) mbar_init(smem_u32(&colFull[b * 4 + k]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // (whole warp walks the loop so it stays converged; lane 0 issues)
    if (nblk > 0) {
      const uint32_t fa = smem_u32(&bars[0]);
      if (lane == 0) {
        mbar_expect_tx(fa, 2 * kHdPackBytes);
        const uint8_t* a0 = P.a_pack + static_cast<int64_t>(row_base / kHdBlockRows) * kHdPackBytes;
        bulk_g2s(smem_u32(sA), a0, kHdPackBytes, fa);
        bulk_g2s(smem_u32(sA + kHdPackBytes), a0 + kHdPackBytes, kHdPackBytes, fa);
      }
      int64_t rk = P.tile_rptr[item.y];  // range walker: position -> column
      int32_t racc = 0;
      for (int t = 0; t < nblk; ++t) {
        const int s = t % L::kStages, ns = t / L::kStages, buf = t & 1;
        const int32_t pos = (pb0 + t) * kHdBlockRows;
        int2 rg = P.ranges[rk];
        while (pos >= racc + (rg.y - rg.x)) {
          racc += rg.y - rg.x;
          rg = P.ranges[++rk];
        }
        const int cblk = (rg.x + (pos - racc)) / kHdBlockRows;
        if (ns > 0) mbar_wait(smem_u32(&emptyB[s]), (ns - 1) & 1);
        if (lane == 0) {
          const uint32_t fb = smem_u32(&fullB[s]);
          mbar_expect_tx(fb, kHdPackBytes);
          bulk_g2s(smem_u32(sB + s * kHdPackBytes),
                   P.b_pack + static_cast<int64_t>(cblk) * kHdPackBytes, kHdPackBytes, fb);
        }
        // column constants (and factors) of block t into ring slot buf once
        // the epilogue released it (block t - 2)
        if (t >= 2) mbar_wait(smem_u32(&tmemEmpty[buf]), ((t >> 1) - 1) & 1);
        if (lane == 0) {
          ring_blk[buf] = cblk;  // published by the arrive below (release)
          const uint32_t fc = smem_u32(&cFull[buf]);
          mbar_expect_tx(fc, L::kRing * 4);
          float* slot = cring + buf * L::kRing;
          bulk_g2s(smem_u32(slot), P.col_c + static_cast<int64_t>(cblk) * 128, 128 * 4, fc);
          if (kSym)
            bulk_g2s(smem_u32(slot + 128), P.col_c2 + static_cast<int64_t>(cblk) * 128, 128 * 4,
                     fc);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    if (nblk > 0) {
      mbar_wait(smem_u32(&bars[0]), 0);
      for (int t = 0; t < nblk; ++t) {
        const int s = t % L::kStages, ns = t / L::kStages, buf = t & 1;
        mbar_wait(smem_u32(&fullB[s]), ns & 1);
        if (t >= 2) mbar_wait(smem_u32(&tmemEmpty[buf]), ((t >> 1) - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t b_hi = smem_u32(sB + s * kHdPackBytes);
          const uint32_t b_lo = b_hi + kHdBlockBytes;
          for (int h = 0; h < 2; ++h) {
            const uint32_t d = tmem + buf * 256 + h * 128;
            const uint32_t a_hi = smem_u32(sA + h * kHdPackBytes);
            const uint32_t a_lo = a_hi + kHdBlockBytes;
            const uint32_t as[3] = {a_hi, a_hi, a_lo}, bs[3] = {b_hi, b_lo, b_hi};
            for (int c = 0; c < 3; ++c)
              for (int k = 0; k < kHdK / 16; ++k)
                umma_f16(d, umma_desc(as[c] + k * 32), umma_desc(bs[c] + k * 32), kHdIdesc,
                         (c | k) ? 1u : 0u);
          }
          umma_commit(smem_u32(&emptyB[s]));     // smem stage free
          umma_commit(smem_u32(&tmemFull[buf]));  // accumulator ready
        }
        __syncwarp();
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // warp = (TMEM lane quarter q, column quarter cq): rows q*32 + lane of
    // both M halves (two TMEM loads of the same lanes), 32 columns per block
    const int e = warp - 2;                   // 0..15
    const int q = warp & 3;                   // TMEM lane quarter (hardware: warp % 4)
    const int cq = e >> 2;                    // column quarter of the 128-column block
    const int row_end = P.tile_start[item.y + 1];
    const int lr0 = q * 32 + lane, lr1 = 128 + lr0;  // local rows
    const float k2 = P.inv_eps_ln2 * (1.f / (kHdScale * kHdScale));
    const int mid = (row_base + row_end) >> 1;
    const float est_mid = (kSym && P.row_est) ? P.row_est[mid] : 0.f;
    float rr[2], wr[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int row = row_base + (hh ? lr1 : lr0);
      const bool ok = row < row_end;
      const float est = (P.row_est && ok) ? P.row_est[row] : 0.f;
      const float xsq = ok ? P.row_sq[row] : 0.f;
      rr[hh] = ok ? est * P.inv_lam_eps_ln2 - 0.5f * xsq * P.inv_eps_ln2
                  : __int_as_float(0xff800000);
      // evaluate-once: column-sum row factor a_i 2^{-ell (est_i - est_mid)}
      wr[hh] = (kSym && ok) ? exp2f(P.row_lw2[row] - P.ell * (est - est_mid)) : 0.f;
    }
    const float2 K2 = make_float2(k2, k2);
    const float2 R0 = make_float2(rr[0], rr[0]), R1 = make_float2(rr[1], rr[1]);
    const float2 W0 = make_float2(wr[0], wr[0]), W1 = make_float2(wr[1], wr[1]);
    float* stg = stage_all + e * 1024;        // this warp's 32 x 32 transpose area
    float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
    for (int t = 0; t < nblk; ++t) {
      const int buf = t & 1, n = t >> 1;
      mbar_wait(smem_u32(&cFull[buf]), n & 1);
      mbar_wait(smem_u32(&tmemFull[buf]), n & 1);
      tc_fence_after();
      const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * 256 + cq * 32;
      const float4* cv = reinterpret_cast<const float4*>(cring + buf * L::kRing + cq * 32);
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {  // 16 columns at a time (register budget: 18 warps)
      float v0[16], v1[16];
      tmem_ld16(base + sub * 16, v0);
      tmem_ld16(base + 128 + sub * 16, v1);
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4) {
        const int k = sub * 16 + kk;
        const float4 cc = cv[k >> 2];
        const float2 ca = make_float2(cc.x, cc.y), cb = make_float2(cc.z, cc.w);
        const float2 a0 = __ffma2_rn(K2, make_float2(v0[kk], v0[kk + 1]), __fadd2_rn(ca, R0));
        const float2 b0 = __ffma2_rn(K2, make_float2(v0[kk + 2], v0[kk + 3]), __fadd2_rn(cb, R0));
        const float2 a1 = __ffma2_rn(K2, make_float2(v1[kk], v1[kk + 1]), __fadd2_rn(ca, R1));
        const float2 b1 = __ffma2_rn(K2, make_float2(v1[kk + 2], v1[kk + 3]), __fadd2_rn(cb, R1));
        const float2 xa0 = make_float2(ex2_approx(a0.x), ex2_approx(a0.y));
        const float2 xb0 = make_float2(ex2_approx(b0.x), ex2_approx(b0.y));
        const float2 xa1 = make_float2(ex2_approx(a1.x), ex2_approx(a1.y));
        const float2 xb1 = make_float2(ex2_approx(b1.x), ex2_approx(b1.y));
        s0 = __fadd2_rn(s0, __fadd2_rn(xa0, xb0));
        s1 = __fadd2_rn(s1, __fadd2_rn(xa1, xb1));
        if (kSym) {  // both rows' weighted terms, chunk k/4 of this lane's staged row
          const float2 ta = __ffma2_rn(W1, xa1, __fmul2_rn(W0, xa0));
          const float2 tb = __ffma2_rn(W1, xb1, __fmul2_rn(W0, xb0));
          *reinterpret_cast<float4*>(stg + lane * 32 + (((k >> 2) ^ (lane & 7)) << 2)) =
              make_float4(ta.x, ta.y, tb.x, tb.y);
        }
      }
      }
      if (!kSym) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tmemEmpty[buf]));
        continue;
      }
      tc_fence_before();  // TMEM reads of this block are done
      // column sums of the warp's 64 rows: lane = chunk g = lane & 7 (columns
      // 4g..4g+3) over staged rows (lane >> 3) + 4i, then lane bits 3, 4
      {
        const int g = lane & 7;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rw = (lane >> 3) + 4 * i;
          const float4 b4 = *reinterpret_cast<const float4*>(stg + rw * 32 + ((g ^ (rw & 7)) << 2));
          a.x += b4.x;
          a.y += b4.y;
          a.z += b4.z;
          a.w += b4.w;
        }
        {
          const bool up = lane & 8;
          const float sx = up ? a.x : a.z, sy = up ? a.y : a.w;
          const float kx = up ? a.z : a.x, ky = up ? a.w : a.y;
          a.x = kx + __shfl_xor_sync(0xffffffffu, sx, 8);
          a.y = ky + __shfl_xor_sync(0xffffffffu, sy, 8);
        }
        {
          const bool up = lane & 16;
          const float sx = up ? a.x : a.y, kx = up ? a.y : a.x;
          a.x = kx + __shfl_xor_sync(0xffffffffu, sx, 16);
        }
        const int colw = 4 * g + ((lane >> 3) & 1) * 2 + ((lane >> 4) & 1);
        colacc[((buf * 4 + cq) * 4 + q) * 32 + colw] = a.x;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&colFull[buf * 4 + cq]));
      if (q == 0) {
        // the column quarter's writer: waits for its 4 lane-quarter warps,
        // combines in a fixed order, applies the column factor
        // 2^{ell (h_j - est_mid) - log2 w_j} and writes the CTA partial.  It
        // releases the TMEM/ring slot only afterwards, so no warp can reach
        // block t + 2 (and overwrite colacc[buf] or the ring) before.
        mbar_wait(smem_u32(&colFull[buf * 4 + cq]), n & 1);
        const float fac = exp2f(cring[buf * L::kRing + 128 + cq * 32 + lane] - P.ell * est_mid);
        const float* ca = colacc + (buf * 4 + cq) * 4 * 32 + lane;
        const float sum = ((ca[0] + ca[32]) + ca[64]) + ca[96];
        const int col = ring_blk[buf] * kHdBlockRows + cq * 32 + lane;
        const int32_t pos = (pb0 + t) * kHdBlockRows + cq * 32 + lane;
        if (col < P.n_cols) P.colpart[P.tile_slot[item.y] + pos] = sum * fac;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tmemEmpty[buf]));
    }
    // the four column quarters of a row: fixed order
    rowacc[cq * kTileRows + lr0] = s0.x + s0.y;
    rowacc[cq * kTileRows + lr1] = s1.x + s1.y;
    named_bar(1, 32 * kHdEpiWarps);
    if (cq == 0) {
      float* out = G.part + static_cast<int64_t>(it) * kTileRows;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int l = hh ? lr1 : lr0;
        out[l] = ((rowacc[l] + rowacc[kTileRows + l]) + rowacc[2 * kTileRows + l]) +
                 rowacc[3 * kTileRows + l];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Column constants of one problem (per scale): c_j = log2 w_j + (h_j - |y_j|^2
// / 2) / (eps ln2), -inf for padding columns up to the 128-column block; and,
// for evaluate-once groups (c2 != null), the column factors' exponent
// c2_j = ell h_j - log2 w_j.
__global__ void hd_colconst_kernel(const float* lw2, const float* h, const float* sq, float inv,
                                   float ell, int32_t n, int32_t npad, float* out, float* out2) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= npad) return;
  out[j] = j < n ? lw2[j] + (h[j] - 0.5f * sq[j]) * inv : __int_as_float(0xff800000);
  // zero-weight columns (padding) feed no column sum: factor 2^-inf = 0
  if (out2) out2[j] = (j < n && lw2[j] > -INFINITY) ? ell * h[j] - lw2[j] : -INFINITY;
}

cudaError_t hd_colconst(const Problem& P, float* out, float* out2, cudaStream_t st) {
  const int32_t npad = static_cast<int32_t>(hd_padded(P.n_cols));
  ++g_launches;
  hd_colconst_kernel<<<(npad + 255) / 256, 256, 0, st>>>(P.col_lw2, P.col_h, P.col_sq,
                                                         P.inv_eps_ln2, P.ell, P.n_cols, npad,
                                                         out, out2);
  return cudaGetLastError();
}

// Column totals of a dense evaluate-once problem: column j sums the partial
// of every row tile of [t0, t1) that owns it (self: tiles ending at or
// before j), in tile order, float64.
// (blockIdx.y = the problem of a grouped launch)
__global__ void hd_colsum_kernel(const __grid_constant__ DenseColSumGroup g) {
  const DenseColSum& a = g.c[blockIdx.y];
  const float* colpart = a.colpart;
  const int64_t* tslot = a.tslot;
  const int32_t* ts = a.ts;
  const int32_t t0 = a.t0, t1 = a.t1, self = a.self, n_cols = a.n_cols;
  float* tot = a.tot;
  double* acc = a.acc;
  const int first = a.first, last = a.last;
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_cols) return;
  int32_t te = t1;  // self: tiles that end at or before j (ts ascending)
  if (self) {
    int32_t lo = t0, hi = t1;  // first t in [t0, t1) with ts[t + 1] > j
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (ts[mid + 1] > j) hi = mid; else lo = mid + 1;
    }
    te = lo;
  }
  // 8 independent loads per step, added in tile order (bitwise the plain loop)
  auto term = [&](int32_t t) {
    return __ldg(colpart + tslot[t] + (j - (self ? ts[t] : 0)));
  };
  double s = (acc && !first) ? acc[j] : 0.0;  // running total of earlier batches
  int32_t t = t0;
  for (; t + 8 <= te; t += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = term(t + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += static_cast<double>(v[u]);
  }
  for (; t < te; ++t) s += static_cast<double>(term(t));
  if ((last || !acc) && tot) tot[j] = static_cast<float>(s);
  else acc[j] = s;  // (tot null: multi-rank float64 exchange, sym_colsum_kernel)
}

cudaError_t hd_colsum_group(const DenseColSum* c, int n, cudaStream_t st) {
  DenseColSumGroup g{};
  int32_t mx = 0;
  for (int k = 0; k < n; ++k) {
    g.c[k] = c[k];
    mx = max(mx, c[k].n_cols);
  }
  g.n = n;
  if (n <= 0 || mx <= 0) return cudaSuccess;
  ++g_launches;
  hd_colsum_kernel<<<dim3((mx + 255) / 256, n), 256, 0, st>>>(g);
  return cudaGetLastError();
}

// Exact online-max LSE for rows the fixed-reference path rejected (float32,
// CUDA cores), high-dimensional variant of softmin_fallback.
__global__ void softmin_hd_fallback(const __grid_constant__ Group G, int d) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int cnt = min(*G.fb_count, G.fb_cap);
  for (int qq = warp; qq < cnt; qq += nwarps) {
    const int4 pr = G.fb_list[qq];
    const Problem& P = G.P[pr.x];
    const int r = pr.y;
    const float* xr = P.row_f + static_cast<int64_t>(r) * kHdK;
    float m = -INFINITY, s = 0.f;
    for (int j = lane; j < P.n_cols; j += 32) {
      const float* yr = P.col_f + static_cast<int64_t>(j) * kHdK;
      float c = 0.f;
      for (int k = 0; k < d; ++k) {
        const float t = xr[k] - yr[k];
        c = fmaf(t, t, c);
      }
      const float z = P.col_lw2[j] + (P.col_h[j] - 0.5f * c) * P.inv_eps_ln2;
      if (z > m) { s = s * exp2f(m - z) + 1.f; m = z; }
      else s += exp2f(z - m);
    }
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * exp2f(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * exp2f(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      const float est = P.row_est ? P.row_est[r] : 0.f;
      const float ft = -P.lam_eps * kLn2 * (m + log2f(s));
      store_potential(G, P.row_out, r, (1.f - P.mixw) * est + P.mixw * ft);
    }
  }
}

__global__ void hd_weights_kernel(const double* w, int64_t n, float* lw2, double* w64) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  lw2[i] = __double2float_rn(log2(w[i]));
  w64[i] = w[i];
}

cudaError_t hd_weights(const double* w, int64_t n, float* lw2, double* w64, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  hd_weights_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(w, n, lw2, w64);
  return cudaGetLastError();
}

cudaError_t launch_softmin_hd(const Group& g, int d, int n_sm, bool sym, cudaStream_t st) {
  (void)d;
  (void)n_sm;
  if (g.n_items <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(softmin_hd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(HdSmem<false>::kTotal));
    cudaFuncSetAttribute(softmin_hd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(HdSmem<true>::kTotal));
    attr = true;
  }
  ++g_launches;
  if (sym)
    softmin_hd_kernel<true><<<g.n_items, kHdThreads, HdSmem<true>::kTotal, st>>>(g);
  else
    softmin_hd_kernel<false><<<g.n_items, kHdThreads, HdSmem<false>::kTotal, st>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_fallback_hd(const Group& g, int d, int n_sm, cudaStream_t st) {
  ++g_launches;
  softmin_hd_fallback<<<n_sm, 256, 0, st>>>(g, d);
  return cudaGetLastError();
}

}  // namespace msot_dev
