// gemm_tc.cu -- tcgen05/TMEM/TMA GEMM kernels (sm_100a), see gemm_tc.cuh.
//
// CTA = 128 threads, one 128 x BN output tile (cta_group::1, UMMA M = 128):
//   warp 0 lane 0 : TMA producer   (cp.async.bulk.tensor -> S-stage smem ring, mbarrier tx)
//   warp 1 lane 0 : MMA issuer     (tcgen05.mma.kind::tf32, 4 x K=8 per 32-wide k-block,
//                                    tcgen05.commit -> frees the smem stage)
//   warps 2..5    : (3xTF32 only; the CTA then has 192 threads) split each landed stage in
//                   place into hi = x rounded to
//                   the nearest TF32 value and lo = (x - hi) rounded to TF32 in a second
//                   buffer, fence.proxy.async, arrive; the MMA thread then issues
//                   A_lo B_hi + A_hi B_lo + A_hi B_hi per k-slice (FP32-grade products: the
//                   dropped A_lo B_lo and the rounding of lo are <= ~2^-23 |a||b| each)
//   warps 0..3    : epilogue       (tcgen05.ld 32x32b: warp w owns TMEM lanes 32(w%4)..+31,
//   (3xTF32: 2..5)                   i.e. tile rows; functor applied per element)
// Shared-memory layouts are the canonical UMMA SWIZZLE_128B layouts produced directly by
// TMA with CU_TENSOR_MAP_SWIZZLE_128B:
//   K-major  : [rows][128 B] (32 fp32 of K per row), 8-row atoms 1024 B apart (SBO)
//   MN-major : boxes of [32 k-rows][128 B] (32 fp32 of M/N), boxes 4096 B apart (LBO),
//              SWIZZLE_128B_BASE32B (TMA SWIZZLE_128B_ATOM_32B): 4-k-row atoms 512 B apart (SBO)
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

#include "gemm_tc.cuh"

namespace ng {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;        // fp32 elements per 128-byte swizzle row = one k-block
constexpr int kStages = 8;     // barrier slots; the ring depth used is tc_stages() (<= kStages)

// Ring depth: 4 unless NG_TUNE_TC_STAGES (tuning knob, 1..8) says otherwise.
int tc_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NG_TUNE_TC_STAGES");
    v = e ? std::max(1, std::min(kStages, atoi(e))) : 4;
  }
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Round to the nearest TF32 value (cvt.rna: 10 explicit mantissa bits, low 13 bits zero), so
// the tensor core reads it exactly: hi = rna(x), lo = rna(x - hi) (x - hi is exact).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// Shared-memory matrix descriptor, sm100 version field = 1.  layout 2 = SWIZZLE_128B (K-major
// operands), layout 1 = SWIZZLE_128B_BASE32B (the only MN-major layout for 32-bit types:
// 128-byte rows, 32-byte granules XOR-swizzled over 4-row / 512-byte atoms).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// K-major SW128: 8-row atoms 1024 B apart; k-slice j of the 32-wide block starts 32j bytes in.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile, int k) { return smem_desc(tile + k * 32, 16, 1024, 2); }
// MN-major SW128_BASE32B: 32-element MN chunks (boxes of 32 k-rows) 4096 B apart (LBO),
// 4-k-row atoms 512 B apart (SBO); k-slice j (8 k-rows) starts 1024j bytes in.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile, int k) { return smem_desc(tile + k * 1024, 4096, 512, 1); }

// Instruction descriptor: D f32, A/B tf32, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// One 128 x BN output tile: rows m0.., columns n0.., k-blocks kb0 .. kb0+nkb-1.  ntile /
// ztile are the column-tile and split indices used by the NGAPPLY / PARTIAL epilogues.
template <int BN, bool AK, bool BKM, int EPI, bool S3>
__device__ __forceinline__ void tc_tile(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int m0, int n0,
                                        int kb0, int nkb, int ntile, int ztile, const TcEpilogue& epi,
                                        int nstages) {
  // S3: 3xTF32 -- each stage holds [A | B] as landed (then hi parts) and [A_lo | B_lo]
  constexpr uint32_t A_BYTES = kBM * kBK * 4, B_BYTES = BN * kBK * 4, HALF = A_BYTES + B_BYTES;
  constexpr uint32_t STAGE = S3 ? 2 * HALF : HALF;
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));   // power of 2
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned ring (SWIZZLE_128B atoms); pointer arithmetic keeps the shared space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t split_bar[S3 ? kStages : 1];
  __shared__ __align__(8) uint64_t accum_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // epilogue warps: 0..3, or 2..5 with 3xTF32 (warps 2..5 also split the stages); a warp
  // reaches TMEM lanes 32 (warp % 4) .. + 31 only
  constexpr int EW0 = S3 ? 2 : 0;
  const bool epi_warp = warp >= EW0;
  const int q4 = warp & 3;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmB)) : "memory");
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      if (S3) mbar_init(&split_bar[s], 128);
    }
    mbar_init(&accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  pdl_trigger();
  pdl_wait();   // operands and the RMW tile may come from the previous kernel on the stream

  // Read-modify-write epilogues: the old C tile does not depend on the MMA, so every
  // thread loads its row of it now (registers) and the HBM latency overlaps the mainloop.
  constexpr bool RMW = EPI == TC_EPI_AXPY || EPI == TC_EPI_NGAPPLY;
  constexpr int CW = BN >= 32 ? 32 : 16;
  const int row = m0 + q4 * 32 + lane;
  float* __restrict__ cbase = epi.C + (EPI == TC_EPI_PARTIAL ? (int64_t)ztile * epi.zstride : 0);
  float* __restrict__ crow = cbase + (int64_t)row * epi.ldc;
  // coalesced (STORE / PARTIAL / PNORM) epilogue layout: lanes per row, rows per pass
  constexpr int LPR = CW / 4, RPP = 32 / LPR, NP = 32 / RPP;
  const int rr = lane / LPR, cc = (lane % LPR) * 4;
  const int wrow0 = m0 + q4 * 32;
  float oldv[RMW ? BN : 1];
  if (RMW && epi_warp) {
#pragma unroll
    for (int c = 0; c < BN / CW; ++c) {
      const int nb = n0 + c * CW;
      const bool full = row < M && (nb + CW <= N) && ((reinterpret_cast<uintptr_t>(crow + nb) & 15) == 0);
      if (full) {
#pragma unroll
        for (int j = 0; j < CW; j += 4) {
          const float4 o = *reinterpret_cast<const float4*>(crow + nb + j);
          oldv[c * CW + j] = o.x; oldv[c * CW + j + 1] = o.y; oldv[c * CW + j + 2] = o.z; oldv[c * CW + j + 3] = o.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) oldv[c * CW + j] = (row < M && nb + j < N) ? crow[nb + j] : 0.f;
      }
    }
  }

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(&empty_bar[s], ph ^ 1u);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      mbar_expect_tx(&full_bar[s], HALF);
      const int kc = (kb0 + i) * kBK;
      if (AK) {
        tma_load_2d(sa, tmA, kc, m0, &full_bar[s]);
      } else {
#pragma unroll
        for (int j = 0; j < kBM / 32; ++j) tma_load_2d(sa + j * 4096, tmA, m0 + 32 * j, kc, &full_bar[s]);
      }
      if (BKM) {
        tma_load_2d(sb, tmB, kc, n0, &full_bar[s]);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) tma_load_2d(sb + j * 4096, tmB, n0 + 32 * j, kc, &full_bar[s]);
      }
      if (++s == nstages) { s = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    constexpr uint32_t idesc = idesc_tf32(kBM, BN, !AK, !BKM);
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(S3 ? &split_bar[s] : &full_bar[s], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int k = 0; k < kBK / 8; ++k) {
        const uint64_t da = AK ? desc_kmajor(sa, k) : desc_mnmajor(sa, k);
        const uint64_t db = BKM ? desc_kmajor(sb, k) : desc_mnmajor(sb, k);
        if (S3) {
          const uint64_t dal = AK ? desc_kmajor(sa + HALF, k) : desc_mnmajor(sa + HALF, k);
          const uint64_t dbl = BKM ? desc_kmajor(sb + HALF, k) : desc_mnmajor(sb + HALF, k);
          mma_tf32(tmem, dal, db, idesc, (i > 0 || k > 0) ? 1u : 0u);   // small terms first
          mma_tf32(tmem, da, dbl, idesc, 1u);
          mma_tf32(tmem, da, db, idesc, 1u);
        } else {
          mma_tf32(tmem, da, db, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
      }
      umma_commit(&empty_bar[s]);
      if (++s == nstages) { s = 0; ph ^= 1u; }
    }
    umma_commit(&accum_bar);
  } else if (S3 && warp >= 2) {
    // ---------------- 3xTF32 split (warps 2-5): hi in place, lo = x - hi beside it
    const int t = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(&full_bar[s], ph);
      float4* hi = reinterpret_cast<float4*>(smem + s * STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + HALF);
#pragma unroll 4
      for (int q = t; q < (int)(HALF / 16); q += 128) {
        const float4 x = hi[q];
        const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        hi[q] = h;
        lo[q] = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z), tf32_rna(x.w - h.w));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
      mbar_arrive(&split_bar[s]);
      if (++s == nstages) { s = 0; ph ^= 1u; }
    }
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> global (row per thread)
  // Warp w owns TMEM lanes (tile rows) 32w..32w+31.  Chunks of 32 columns (two tcgen05.ld):
  // each thread moves one full 128-byte line of its row per chunk with 8 independent
  // 16-byte accesses (all loads of a read-modify-write chunk are issued first).
  if (epi_warp) {
  mbar_wait(&accum_bar, 0);
  tc_fence_after();
  __syncwarp();
  if constexpr (EPI == TC_EPI_PNORM) {
    // Z row in 80-column halves (8 groups of 10 each) and the group 2-norms
    static_assert(BN % 80 == 0, "p-norm epilogue: tiles of whole 80-column blocks");
    float* yrow = epi.y + (int64_t)row * epi.ldy;
#pragma unroll 1
    for (int hh = 0; hh < BN / 80; ++hh) {
      const int nh = n0 + hh * 80;
      float acc[80];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(hh * 80 + c * 16), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c * 16 + j] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      }
      // Z store, coalesced: 16-column chunks through a per-warp shared-memory transpose (the
      // ring is idle), 4 lanes x 16 bytes per row, 8 rows per warp instruction
      {
        float* sc = reinterpret_cast<float*>(smem) + q4 * (32 * 17);
        const int rr = lane >> 2, cc = (lane & 3) * 4;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
#pragma unroll
          for (int j = 0; j < 16; ++j) sc[lane * 17 + j] = acc[c * 16 + j];
          __syncwarp();
          const int gc = nh + c * 16 + cc;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int lr = p * 8 + rr, r = m0 + q4 * 32 + lr;
            const float* s4 = sc + lr * 17 + cc;
            const float4 v = make_float4(s4[0], s4[1], s4[2], s4[3]);
            if (r < M && gc < N) {
              float* dst = cbase + (int64_t)r * epi.ldc + gc;
              if (gc + 4 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                *reinterpret_cast<float4*>(dst) = v;
              } else {
                dst[0] = v.x;
                if (gc + 1 < N) dst[1] = v.y;
                if (gc + 2 < N) dst[2] = v.z;
                if (gc + 3 < N) dst[3] = v.w;
              }
            }
          }
          __syncwarp();
        }
      }
      if (row < M && nh < N) {
        const int g0 = nh / 10;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float sq = 0.f;
#pragma unroll
          for (int q = 0; q < 10; ++q) sq = fmaf(acc[g * 10 + q], acc[g * 10 + q], sq);
          if (nh + g * 10 + 10 <= N) yrow[g0 + g] = sqrtf(sq);
        }
        if (nh + 80 >= N) {   // last column block: bias input and the zero padding
          const int dp = N / 10;
          yrow[dp] = 1.f;
          for (int c = dp + 1; c < epi.ldy; ++c) yrow[c] = 0.f;
        }
      }
    }
  } else if constexpr (RMW) {
  // read-modify-write (AXPY, NGAPPLY): thread = row, old C already in registers (measured
  // faster than the coalesced transpose below for these two)
  const float scale = (EPI == TC_EPI_AXPY) ? __ldg(epi.scale) : 0.f;
  float xx = 0.f, pp = 0.f;   // TC_EPI_NGAPPLY row partial sums over this tile's columns
#pragma unroll
  for (int c = 0; c < BN / CW; ++c) {
    float acc[CW];
    {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(c * CW), v);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      if (CW == 32) {
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(c * CW + 16), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[16 + j] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      }
    }
    const int nb = n0 + c * CW;
    if (row < M && nb < N) {
      const bool full = (nb + CW <= N) && ((reinterpret_cast<uintptr_t>(crow + nb) & 15) == 0);
      if (EPI == TC_EPI_STORE || EPI == TC_EPI_PARTIAL) {
        if (full) {
#pragma unroll
          for (int j = 0; j < CW; j += 4)
            *reinterpret_cast<float4*>(crow + nb + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (nb + j < N) crow[nb + j] = acc[j];
        }
      } else {
        const float* old = oldv + (RMW ? c * CW : 0);
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          if (EPI == TC_EPI_AXPY) {
            acc[j] = fmaf(scale, acc[j], old[j]);
          } else {   // TC_EPI_NGAPPLY: x_hat = x - (H W)  (eqn:hatxt:compute:2), row norms
            const float xn = old[j] - acc[j];
            xx = fmaf(old[j], old[j], xx);
            pp = fmaf(xn, xn, pp);
            acc[j] = xn;
          }
        }
        if (full) {
#pragma unroll
          for (int j = 0; j < CW; j += 4)
            *reinterpret_cast<float4*>(crow + nb + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (nb + j < N) crow[nb + j] = acc[j];
        }
      }
    }
  }
  if (EPI == TC_EPI_NGAPPLY && row < M) {
    epi.xx[(int64_t)ntile * epi.part_ld + row] = xx;
    epi.pp[(int64_t)ntile * epi.part_ld + row] = pp;
  }
  } else {
  // STORE / PARTIAL, coalesced: each warp moves its 32 rows x CW columns from TMEM (thread =
  // row) through a padded shared-memory transpose (the ring is idle once accum_bar fired) so
  // a warp instruction covers whole 128-byte row segments (LPR lanes x 16 bytes per row)
  // instead of 32 rows x 16 bytes.
  float* sc = reinterpret_cast<float*>(smem) + q4 * (32 * 33);
#pragma unroll 1
  for (int c = 0; c < BN / CW; ++c) {
    {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(c * CW), v);
#pragma unroll
      for (int j = 0; j < 16; ++j) sc[lane * 33 + j] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      if (CW == 32) {
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(c * CW + 16), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) sc[lane * 33 + 16 + j] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      }
    }
    __syncwarp();
    const int gc = n0 + c * CW + cc;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int lr = p * RPP + rr, r = wrow0 + lr;
      const float* s4 = sc + lr * 33 + cc;
      const float4 v = make_float4(s4[0], s4[1], s4[2], s4[3]);
      if (r < M && gc < N) {
        float* dst = cbase + (int64_t)r * epi.ldc + gc;
        if (gc + 4 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          *reinterpret_cast<float4*>(dst) = v;
        } else {
          dst[0] = v.x;
          if (gc + 1 < N) dst[1] = v.y;
          if (gc + 2 < N) dst[2] = v.z;
          if (gc + 3 < N) dst[3] = v.w;
        }
      }
    }
    __syncwarp();
  }
  }   // EPI != TC_EPI_PNORM
  }   // epi_warp
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int BN, bool AK, bool BKM, int EPI, bool S3>
__global__ void __launch_bounds__(S3 ? 192 : 128)
tc_gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, int kb_per_split, TcEpilogue epi, int nstages) {
  const int kb_total = (K + kBK - 1) / kBK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(kb_total, kb0 + kb_per_split) - kb0);
  tc_tile<BN, AK, BKM, EPI, S3>(&tmA, &tmB, M, N, blockIdx.y * kBM, blockIdx.x * BN, kb0, nkb, blockIdx.x,
                                blockIdx.z, epi, nstages);
}

// Grouped launch: problem g owns tiles [tile_begin, tile_begin + mt*nt*splits); each tile
// (z, m, n) of it is one CTA.  Problems share BN, operand majors and epilogue kind.
template <int BN, bool AK, bool BKM, int EPI, bool S3>
__global__ void __launch_bounds__(S3 ? 192 : 128) tc_gemm_tf32_grouped_kernel(const __grid_constant__ TcGroup grp) {
  int g = 0;
  while (g + 1 < grp.count && (int)blockIdx.x >= grp.p[g + 1].tile_begin) ++g;
  const TcProblem& P = grp.p[g];
  const int local = (int)blockIdx.x - P.tile_begin;
  const int nt = (P.N + BN - 1) / BN, mt = (P.M + kBM - 1) / kBM;
  const int ntile = local % nt, mtile = (local / nt) % mt, z = local / (nt * mt);
  const int kb_total = (P.K + kBK - 1) / kBK;
  const int kb0 = z * P.kbps;
  const int nkb = max(0, min(kb_total, kb0 + P.kbps) - kb0);
  tc_tile<BN, AK, BKM, EPI, S3>(&P.tmA, &P.tmB, P.M, P.N, mtile * kBM, ntile * BN, kb0, nkb, ntile, z, P.epi,
                                grp.nstages);
}

// Persistent grouped weight update C += (*scale) A B (TC_EPI_AXPY, both operands MN-major,
// 128 x 128 tiles, TF32): one CTA per SM walks tiles blockIdx.x, +gridDim.x, ...  Warp 0
// lane 0 streams every tile's k-blocks through one TMA ring, warp 1 lane 0 issues the MMAs
// into one of TWO TMEM accumulators (256 columns), and warps 2..5 drain the other one (the
// read-modify-write of the previous tile, its old C prefetched while the MMAs run), so the
// epilogue of tile i overlaps the mainloop of tile i + 1.
__global__ void __launch_bounds__(192) tc_axpy_persistent_kernel(const __grid_constant__ TcGroup grp, int tiles) {
  constexpr int BN = 128;
  constexpr uint32_t A_BYTES = kBM * kBK * 4, B_BYTES = BN * kBK * 4, STAGE = A_BYTES + B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t acc_full[2];
  __shared__ __align__(8) uint64_t acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nstages = grp.nstages;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < nstages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  pdl_trigger();
  pdl_wait();

  // tile -> (problem, m tile, n tile)
  auto locate = [&](int t, int& g, int& m0, int& n0) {
    g = 0;
    while (g + 1 < grp.count && t >= grp.p[g + 1].tile_begin) ++g;
    const TcProblem& P = grp.p[g];
    const int local = t - P.tile_begin, nt = (P.N + BN - 1) / BN;
    n0 = (local % nt) * BN;
    m0 = (local / nt) * kBM;
  };
  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: every k-block of every tile of this CTA
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int g, m0, n0;
        locate(t, g, m0, n0);
        const TcProblem& P = grp.p[g];
        const int nkb = (P.K + kBK - 1) / kBK;
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sa = smem + s * STAGE;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full_bar[s], STAGE);
          const int kc = i * kBK;
#pragma unroll
          for (int j = 0; j < kBM / 32; ++j) tma_load_2d(sa + j * 4096, &P.tmA, m0 + 32 * j, kc, &full_bar[s]);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) tma_load_2d(sb + j * 4096, &P.tmB, n0 + 32 * j, kc, &full_bar[s]);
          if (++s == nstages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer, accumulators alternating between TMEM columns 0 and 128
      constexpr uint32_t idesc = idesc_tf32(kBM, BN, true, true);
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        int g, m0, n0;
        locate(t, g, m0, n0);
        const int nkb = (grp.p[g].K + kBK - 1) / kBK;
        const int b = it & 1;
        mbar_wait(&acc_empty[b], ((it >> 1) & 1) ^ 1u);   // the epilogue has drained buffer b
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k)
            mma_tf32(acc, desc_mnmajor(sa, k), desc_mnmajor(sb, k), idesc, (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty_bar[s]);
          if (++s == nstages) { s = 0; ph ^= 1u; }
        }
        umma_commit(&acc_full[b]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 (TMEM lane quarter = warp % 4)
    const int q4 = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      int g, m0, n0;
      locate(t, g, m0, n0);
      const TcProblem& P = grp.p[g];
      const int b = it & 1;
      const int row = m0 + q4 * 32 + lane;
      float* crow = P.epi.C + (int64_t)row * P.epi.ldc;
      const float scale = __ldg(P.epi.scale);
      // the old C row segment does not depend on the MMAs: load it before waiting for them
      const bool rowok = row < P.M;
      const bool vec = rowok && (n0 + BN <= P.N) && ((reinterpret_cast<uintptr_t>(crow + n0) & 15) == 0);
      float oldv[BN];
      if (vec) {
#pragma unroll
        for (int j = 0; j < BN; j += 4) {
          const float4 o = *reinterpret_cast<const float4*>(crow + n0 + j);
          oldv[j] = o.x; oldv[j + 1] = o.y; oldv[j + 2] = o.z; oldv[j + 3] = o.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < BN; ++j) oldv[j] = (rowok && n0 + j < P.N) ? crow[n0 + j] : 0.f;
      }
      mbar_wait(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      __syncwarp();
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        const int nb = n0 + c * 32;
        float acc[32];
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * BN + c * 32), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(v[j]);
        tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * BN + c * 32 + 16), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[16 + j] = __uint_as_float(v[j]);
        if (vec) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(crow + nb + 4 * j) = make_float4(
                fmaf(scale, acc[4 * j], oldv[c * 32 + 4 * j]), fmaf(scale, acc[4 * j + 1], oldv[c * 32 + 4 * j + 1]),
                fmaf(scale, acc[4 * j + 2], oldv[c * 32 + 4 * j + 2]), fmaf(scale, acc[4 * j + 3], oldv[c * 32 + 4 * j + 3]));
        } else if (rowok) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (nb + j < P.N) crow[nb + j] = fmaf(scale, acc[j], oldv[c * 32 + j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D fp32 tensor [outer][inner] with row stride ld (elements), box {32, box_outer};
// mn_major selects the 32-byte-atom 128B swizzle (SWIZZLE_128B_ATOM_32B).
ng_status make_tmap(CUtensorMap* out, const float* ptr, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                    bool mn_major) {
  using Key = std::tuple<const float*, int64_t, int64_t, int64_t, int, bool>;
  static std::map<Key, CUtensorMap> cache;
  const Key key{ptr, inner, outer, ld, box_outer, mn_major};
  auto it = cache.find(key);
  if (it != cache.end()) { *out = it->second; return NG_OK; }
  EncodeTiledFn fn = encode_fn();
  NG_REQUIRE(fn != nullptr, NG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  NG_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (ld % 4) == 0, NG_ESHAPE,
             "TMA operand must be 16B aligned with ld % 4 == 0");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    return NG_ECUDA;
  }
  if (cache.size() > 4096) cache.clear();
  cache[key] = m;
  *out = m;
  return NG_OK;
}

inline size_t ring_smem(int bn, int stages, bool s3) {
  return (size_t)stages * (kBM * kBK * 4 + bn * kBK * 4) * (s3 ? 2 : 1) + 1024;
}
// Ring depth for BN, capped by the 227 KB dynamic shared memory limit.
inline int ring_stages(int bn, bool s3) {
  int ns = tc_stages();
  while (ns > 1 && ring_smem(bn, ns, s3) > 227u * 1024u) --ns;
  return ns;
}

template <int BN, bool AK, bool BKM, int EPI, bool S3>
ng_status launch(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int kbps,
                 int splits, const TcEpilogue& epi) {
  static bool attr = false;
  if (!attr) {
    NG_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_tf32_kernel<BN, AK, BKM, EPI, S3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ring_smem(BN, ring_stages(BN, S3), S3)));
    attr = true;
  }
  // Only as many ring stages as k-blocks per tile: short-K tiles leave room for more
  // co-resident CTAs per SM.
  const int ns = std::max(1, std::min(ring_stages(BN, S3), kbps));
  dim3 grid(ceil_div(N, BN), ceil_div(M, kBM), splits);
  NG_CUDA_TRY(launch_pdl(tc_gemm_tf32_kernel<BN, AK, BKM, EPI, S3>, grid, dim3(S3 ? 192 : 128), ring_smem(BN, ns, S3), st, ta,
                         tb, M, N, K, kbps, epi, ns));
  return check_launch("tc_gemm_tf32_kernel");
}

template <int BN, bool AK, bool BKM, bool S3>
ng_status dispatch_epi(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int kbps,
                       int splits, const TcEpilogue& epi) {
  switch (epi.kind) {
    case TC_EPI_STORE: return launch<BN, AK, BKM, TC_EPI_STORE, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
    case TC_EPI_AXPY: return launch<BN, AK, BKM, TC_EPI_AXPY, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
    case TC_EPI_NGAPPLY: return launch<BN, AK, BKM, TC_EPI_NGAPPLY, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
    default: return launch<BN, AK, BKM, TC_EPI_PARTIAL, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
  }
}

template <int BN, bool S3>
ng_status dispatch_major(cudaStream_t st, bool ak, bool bk, const CUtensorMap& ta, const CUtensorMap& tb, int M,
                         int N, int K, int kbps, int splits, const TcEpilogue& epi) {
  if (ak && bk) return dispatch_epi<BN, true, true, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
  if (ak && !bk) return dispatch_epi<BN, true, false, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
  if (!ak && bk) return dispatch_epi<BN, false, true, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
  return dispatch_epi<BN, false, false, S3>(st, ta, tb, M, N, K, kbps, splits, epi);
}

template <bool S3>
ng_status dispatch_bn(cudaStream_t st, int bn, bool ak, bool bk, const CUtensorMap& ta, const CUtensorMap& tb, int M,
                      int N, int K, int kbps, int splits, const TcEpilogue& epi) {
  if (bn == 32) return dispatch_major<32, S3>(st, ak, bk, ta, tb, M, N, K, kbps, splits, epi);
  if (bn == 64) return dispatch_major<64, S3>(st, ak, bk, ta, tb, M, N, K, kbps, splits, epi);
  return dispatch_major<128, S3>(st, ak, bk, ta, tb, M, N, K, kbps, splits, epi);
}

}  // namespace

int tc_splits(int K, int splits) {
  const int kb = std::max(1, ceil_div(K, kBK));
  splits = std::max(1, std::min(splits, kb));
  const int kbps = ceil_div(kb, splits);
  return ceil_div(kb, kbps);
}

ng_status tc_gemm_tf32(cudaStream_t st, int M, int N, int K, const float* A, int64_t lda, bool a_kmajor,
                       const float* B, int64_t ldb, bool b_kmajor, const TcEpilogue& epi, int bn, int splits,
                       int* splits_used, bool split3) {
  NG_REQUIRE(M >= 1 && N >= 1 && K >= 1, NG_ESHAPE, "tc_gemm_tf32: empty problem");
  NG_REQUIRE(bn == 32 || bn == 64 || bn == 128, NG_EINVAL, "tc_gemm_tf32: bn must be 32, 64 or 128");
  const int kb = ceil_div(K, kBK);
  splits = tc_splits(K, splits);
  const int kbps = ceil_div(kb, splits);
  NG_REQUIRE(splits == 1 || epi.kind == TC_EPI_PARTIAL, NG_EINVAL, "split-K needs the partial epilogue");
  if (splits_used) *splits_used = splits;
  CUtensorMap ta, tb;
  if (a_kmajor) NG_TRY(make_tmap(&ta, A, K, M, lda, kBM, false));     // [M][K]
  else NG_TRY(make_tmap(&ta, A, M, K, lda, 32, true));                // [K][M]
  if (b_kmajor) NG_TRY(make_tmap(&tb, B, K, N, ldb, bn, false));      // [N][K]
  else NG_TRY(make_tmap(&tb, B, N, K, ldb, 32, true));                // [K][N]
  if (split3) return dispatch_bn<true>(st, bn, a_kmajor, b_kmajor, ta, tb, M, N, K, kbps, splits, epi);
  return dispatch_bn<false>(st, bn, a_kmajor, b_kmajor, ta, tb, M, N, K, kbps, splits, epi);
}

ng_status tc_gemm_tf32_pnorm(cudaStream_t st, int M, int N, int K, const float* A, int64_t lda, const float* B,
                                  int64_t ldb, float* Z, int64_t ldz, float* Ynext, int64_t ldy, bool split3) {
  NG_REQUIRE(M >= 1 && N >= 10 && K >= 1 && N % 10 == 0 && ldy >= N / 10 + 1, NG_ESHAPE, "tc_gemm_tf32_pnorm: shape");
  const int kb = ceil_div(K, kBK);
  CUtensorMap ta, tb;
  NG_TRY(make_tmap(&ta, A, K, M, lda, kBM, false));
  // 80 or 160 columns (8 or 16 whole groups) per tile (NG_TUNE_FWD_PNORM_BN)
  static const int bn = tune_int("NG_TUNE_FWD_PNORM_BN", 80) == 160 ? 160 : 80;
  NG_TRY(make_tmap(&tb, B, K, N, ldb, bn, false));
  TcEpilogue e;
  e.kind = TC_EPI_PNORM;
  e.C = Z;
  e.ldc = ldz;
  e.y = Ynext;
  e.ldy = ldy;
  if (split3) return launch<80, true, true, TC_EPI_PNORM, true>(st, ta, tb, M, N, K, kb, 1, e);
  if (bn == 160) return launch<160, true, true, TC_EPI_PNORM, false>(st, ta, tb, M, N, K, kb, 1, e);
  return launch<80, true, true, TC_EPI_PNORM, false>(st, ta, tb, M, N, K, kb, 1, e);
}

template <int BN, bool AK, bool BKM, int EPI, bool S3>
ng_status launch_grouped(cudaStream_t st, const TcGroup& grp, int tiles) {
  static bool attr = false;
  if (!attr) {
    NG_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_tf32_grouped_kernel<BN, AK, BKM, EPI, S3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ring_smem(BN, ring_stages(BN, S3), S3)));
    attr = true;
  }
  NG_CUDA_TRY(launch_pdl(tc_gemm_tf32_grouped_kernel<BN, AK, BKM, EPI, S3>, dim3(tiles), dim3(S3 ? 192 : 128),
                         ring_smem(BN, grp.nstages, S3), st, grp));
  return check_launch("tc_gemm_tf32_grouped_kernel");
}

template <bool S3>
ng_status grouped_dispatch(cudaStream_t st, const TcGroup& grp, int tiles, bool a_kmajor, bool b_kmajor, int epi_kind,
                           int bn);

ng_status tc_gemm_tf32_grouped(cudaStream_t st, const TcGroupDesc* desc, int count, bool a_kmajor, bool b_kmajor,
                               int epi_kind, int bn, bool split3) {
  NG_REQUIRE(count >= 1 && count <= kTcGroupMax, NG_EINVAL, "tc_gemm_tf32_grouped: bad problem count");
  NG_REQUIRE(bn == 32 || bn == 64 || bn == 128, NG_EINVAL, "tc_gemm_tf32_grouped: bad bn");
  TcGroup grp;
  std::memset(&grp, 0, sizeof(grp));
  grp.count = count;
  int tiles = 0, kbps_max = 1;
  for (int g = 0; g < count; ++g) {
    const TcGroupDesc& d = desc[g];
    NG_REQUIRE(d.M >= 1 && d.N >= 1 && d.K >= 1, NG_ESHAPE, "tc_gemm_tf32_grouped: empty problem");
    const int kb = ceil_div(d.K, kBK);
    const int sp = tc_splits(d.K, d.splits);
    NG_REQUIRE(sp == 1 || epi_kind == TC_EPI_PARTIAL, NG_EINVAL, "split-K needs the partial epilogue");
    TcProblem& P = grp.p[g];
    if (a_kmajor) NG_TRY(make_tmap(&P.tmA, d.A, d.K, d.M, d.lda, kBM, false));
    else NG_TRY(make_tmap(&P.tmA, d.A, d.M, d.K, d.lda, 32, true));
    if (b_kmajor) NG_TRY(make_tmap(&P.tmB, d.B, d.K, d.N, d.ldb, bn, false));
    else NG_TRY(make_tmap(&P.tmB, d.B, d.N, d.K, d.ldb, 32, true));
    P.M = d.M; P.N = d.N; P.K = d.K;
    P.kbps = ceil_div(kb, sp);
    kbps_max = std::max(kbps_max, P.kbps);
    P.tile_begin = tiles;
    P.epi = d.epi;
    if (d.splits_used) *d.splits_used = sp;
    tiles += ceil_div(d.M, kBM) * ceil_div(d.N, bn) * sp;
  }
  grp.nstages = std::min(ring_stages(bn, split3), kbps_max);
  if (split3) return grouped_dispatch<true>(st, grp, tiles, a_kmajor, b_kmajor, epi_kind, bn);
  return grouped_dispatch<false>(st, grp, tiles, a_kmajor, b_kmajor, epi_kind, bn);
}

template <bool S3>
ng_status grouped_dispatch(cudaStream_t st, const TcGroup& grp, int tiles, bool a_kmajor, bool b_kmajor, int epi_kind,
                           int bn) {
#define NG_GRP(BN_, AK_, BK_, E_) return launch_grouped<BN_, AK_, BK_, E_, S3>(st, grp, tiles)
#define NG_GRP_E(BN_, AK_, BK_)                                         \
  switch (epi_kind) {                                                  \
    case TC_EPI_STORE: NG_GRP(BN_, AK_, BK_, TC_EPI_STORE);            \
    case TC_EPI_AXPY: NG_GRP(BN_, AK_, BK_, TC_EPI_AXPY);              \
    case TC_EPI_NGAPPLY: NG_GRP(BN_, AK_, BK_, TC_EPI_NGAPPLY);        \
    default: NG_GRP(BN_, AK_, BK_, TC_EPI_PARTIAL);                    \
  }
#define NG_GRP_M(BN_)                                                  \
  if (a_kmajor && b_kmajor) { NG_GRP_E(BN_, true, true) }              \
  if (a_kmajor && !b_kmajor) { NG_GRP_E(BN_, true, false) }            \
  if (!a_kmajor && b_kmajor) { NG_GRP_E(BN_, false, true) }            \
  NG_GRP_E(BN_, false, false)
  if (bn == 32) { NG_GRP_M(32) }
  if (bn == 64) { NG_GRP_M(64) }
  NG_GRP_M(128)
#undef NG_GRP_M
#undef NG_GRP_E
#undef NG_GRP
}

ng_status tc_gemm_tf32_axpy_persistent(cudaStream_t st, const TcGroupDesc* desc, int count) {
  NG_REQUIRE(count >= 1 && count <= kTcGroupMax, NG_EINVAL, "tc_gemm_tf32_axpy_persistent: bad problem count");
  constexpr int BN = 128;
  TcGroup grp;
  std::memset(&grp, 0, sizeof(grp));
  grp.count = count;
  int tiles = 0;
  for (int g = 0; g < count; ++g) {
    const TcGroupDesc& d = desc[g];
    NG_REQUIRE(d.M >= 1 && d.N >= 1 && d.K >= 1 && d.epi.kind == TC_EPI_AXPY, NG_EINVAL, "axpy problems only");
    TcProblem& P = grp.p[g];
    NG_TRY(make_tmap(&P.tmA, d.A, d.M, d.K, d.lda, 32, true));   // [K][M]
    NG_TRY(make_tmap(&P.tmB, d.B, d.N, d.K, d.ldb, 32, true));   // [K][N]
    P.M = d.M; P.N = d.N; P.K = d.K; P.kbps = ceil_div(d.K, kBK);
    P.tile_begin = tiles;
    P.epi = d.epi;
    tiles += ceil_div(d.M, kBM) * ceil_div(d.N, BN);
  }
  grp.nstages = ring_stages(BN, false);
  const size_t smem = ring_smem(BN, grp.nstages, false);
  static bool attr = false;
  if (!attr) {
    NG_CUDA_TRY(cudaFuncSetAttribute(tc_axpy_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ring_smem(BN, ring_stages(BN, false), false)));
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  NG_CUDA_TRY(launch_pdl(tc_axpy_persistent_kernel, dim3(std::min(tiles, sms)), dim3(192), smem, st, grp, tiles));
  return check_launch("tc_axpy_persistent_kernel");
}

// Fixed-order reduction of split-K partials: C[m][n] = sum_z part[z][m][n].
__global__ void reduce_partials_kernel(float* __restrict__ C, int64_t ldc, const float* __restrict__ part, int M,
                                       int N, int sp) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < sp; ++z) s += part[(int64_t)z * total + i];
    C[(i / N) * ldc + (i % N)] = s;
  }
}

ng_status reduce_partials_2d(cudaStream_t st, float* C, int64_t ldc, const float* part, int M, int N, int sp) {
  reduce_partials_kernel<<<std::min(4096, ceil_div((int64_t)M * N, 256)), 256, 0, st>>>(C, ldc, part, M, N, sp);
  return check_launch("reduce_partials_kernel");
}

}  // namespace ng

// ------------------------------------------------------------------ C ABI diagnostics

extern "C" ng_status ng_debug_gemm_tf32(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda, int32_t a_kmajor,
                                        const float* B, int64_t ldb, int32_t b_kmajor, float* C, int64_t ldc,
                                        int32_t bn, int32_t splits, void* stream) {
  return ng_debug_gemm_tc(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, C, ldc, bn, splits, 0, stream);
}

extern "C" ng_status ng_debug_gemm_tc(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda, int32_t a_kmajor,
                                      const float* B, int64_t ldb, int32_t b_kmajor, float* C, int64_t ldc,
                                      int32_t bn, int32_t splits, int32_t split3, void* stream) {
  using namespace ng;
  NG_REQUIRE(A && B && C, NG_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  TcEpilogue e;
  if (splits <= 1) {
    e.kind = TC_EPI_STORE;
    e.C = C;
    e.ldc = ldc;
    return tc_gemm_tf32(st, M, N, K, A, lda, a_kmajor != 0, B, ldb, b_kmajor != 0, e, bn, 1, nullptr, split3 != 0);
  }
  const int sp = tc_splits(K, splits);
  float* part = nullptr;
  NG_CUDA_TRY(cudaMallocAsync((void**)&part, sizeof(float) * (size_t)sp * M * N, st));
  e.kind = TC_EPI_PARTIAL;
  e.C = part;
  e.ldc = N;
  e.zstride = (int64_t)M * N;
  ng_status s = tc_gemm_tf32(st, M, N, K, A, lda, a_kmajor != 0, B, ldb, b_kmajor != 0, e, bn, sp, nullptr, split3 != 0);
  if (s == NG_OK) s = reduce_partials_2d(st, C, ldc, part, M, N, sp);
  cudaFreeAsync(part, st);
  return s;
}
