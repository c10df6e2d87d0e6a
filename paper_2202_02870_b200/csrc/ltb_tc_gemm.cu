// 5th-generation tensor-core GEMM (tcgen05 + TMA + TMEM) for FP32 data with
// the 3xTF32 split:  A*B ~= Ahi*Bhi + Ahi*Blo + Alo*Bhi,  hi = x with the low
// 13 mantissa bits cleared (exactly representable in TF32), lo = x - hi.
// Plain TF32 misses the 1e-4 parity bar on the *_L product (SURVEY.md §7
// "hard part 2": 6.3e-4 measured); the split restores ~FP32 accuracy.
//
// C[b] (M x N, row-major, ldc) = A[b] (M x K) * B[b] (K x N), where each
// operand is either K-major (A: M rows of K contiguous; B: N rows of K
// contiguous) or MN-major (A stored K x M; B stored K x N).  This one kernel
// serves the whole f32 *_L product (linalg.py:34-43):
//   forward transform  tube->slice : C(P x NT) = Kron(P x P) * X^T         (A K-major, B K-major)
//   slice GEMM         (K2)        : C_q = Ahat_q * Bhat_q                  (A K-major, B MN-major)
//   inverse transform  slice->tube : C(NT x P) = H^T(NT x P) * Kinv^T       (A MN-major, B K-major)
// with the transform applied as one dense Kronecker matrix (P <= 1024).
//
// Structure (one 128 x BN output tile per CTA, 8 warps):
//   warp 0      TMA producer (one elected lane), 3-stage smem ring, 128B swizzle
//   warp 1      TMEM allocator + MMA issuer (one lane): 3 tcgen05.mma kind::tf32
//               per K=8 step, accumulator in TMEM, tcgen05.commit frees a stage
//   warps 2-3   split converters: in place hi, separate lo buffer, then
//               fence.proxy.async so the tensor core sees the generic writes
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> registers -> global
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "ltb_dispatch.cuh"

namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kStages = 3;
constexpr int kThreads = 384;  // 12 warps: TMA, MMA, 6 split converters, 4 epilogue
constexpr int kConv = 192;     // split-converter threads (warps 2-7)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor (sm100 version bits = 1).  K-major operands use
// SWIZZLE_128B (layout 2, 8-row 1 KB atoms); 32-bit MN-major operands use
// SWIZZLE_128B_BASE32B (layout 1, 4 K-row 512 B atoms), which is what the TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B mode writes.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              bool mn32 = false) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                     // descriptor version (Blackwell)
  d |= (uint64_t)(mn32 ? 1 : 2) << 61;        // SWIZZLE_128B_BASE32B : SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::tf32, D f32, A/B tf32, M = 128, N = BN
__host__ __device__ constexpr uint32_t idesc_tf32(int bn, bool a_mn, bool b_mn) {
  return (1u << 4)                       // D format f32
         | (2u << 7)                     // A format tf32
         | (2u << 10)                    // B format tf32
         | ((a_mn ? 1u : 0u) << 15)      // A major
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(bn >> 3) << 17)   // N >> 3
         | ((uint32_t)(kBM >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%"
      "20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 3xTF32 split of one smem tile (layout-agnostic, elementwise):
//   hi = x with the low 13 mantissa bits cleared (what the tensor core reads from
//        x itself: measured on B200, kind::tf32 truncates fp32 -> tf32, so with
//        raw_hi the fp32 tile is left in place as the hi operand),
//   lo = round-to-nearest-tf32(x - hi), so the tensor core's truncation of lo is
//        exact and the residual error is unbiased.
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_round(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
template <int N16>
__device__ __forceinline__ void split_tile(float4* hi, float4* lo, int ct, int raw_hi) {
#pragma unroll 4
  for (int i = ct; i < N16; i += kConv) {
    const float4 x = hi[i];
    const float4 h = make_float4(tf32_trunc(x.x), tf32_trunc(x.y), tf32_trunc(x.z), tf32_trunc(x.w));
    lo[i] = make_float4(tf32_round(x.x - h.x), tf32_round(x.y - h.y), tf32_round(x.z - h.z), tf32_round(x.w - h.w));
    if (!raw_hi) hi[i] = h;
  }
}

// ------------------------------------------------------------------ kernel
// RB ("resident B"): B is one constant matrix (a transform's Kronecker matrix)
// of at most kRbMaxKt K-blocks, loaded once per CTA together with its
// precomputed lo part, so the pipeline streams and splits only A.
constexpr int kRbMaxKt = 3;

template <int BN, bool A_MN, bool B_MN, int SPLIT, bool RB>
struct TcCfg {
  static constexpr int A_BYTES = kBM * kBK * 4;  // 16 KB
  static constexpr int B_BYTES = BN * kBK * 4;
  static constexpr int NSPLIT = SPLIT == 3 ? 2 : 1;
  static constexpr int STAGE_BYTES = RB ? NSPLIT * A_BYTES : NSPLIT * (A_BYTES + B_BYTES);
  static constexpr int RES_BYTES = RB ? kRbMaxKt * NSPLIT * B_BYTES : 0;
  static constexpr int EPI_BYTES = 4 * 2 * 4096;  // per epilogue warp: two 32 x 32 fp32 swizzled store boxes
  static constexpr int SMEM =
      kStages * STAGE_BYTES + RES_BYTES + 1024 /* align */ + 1024 /* barriers */ + EPI_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static_assert(2 * BN <= 512, "two accumulators must fit in TMEM");
  static_assert(B_BYTES % 1024 == 0 && STAGE_BYTES % 1024 == 0, "1 KB swizzle-atom alignment");
  static_assert(!RB || !B_MN, "resident B is K-major");
};

template <int BN, bool A_MN, bool B_MN, int SPLIT, bool RB>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmC,
                        float* __restrict__ C, int64_t ldc, int64_t sc, int M, int N, int K, int batches,
                        uint32_t mn_lbo, uint32_t mn_sbo, int raw_hi, unsigned long long* dbg, int epi_mode, int ct) {
  // optional timeline instrumentation (CTA 0, %globaltimer ns) for the launch-cost analysis
  auto stamp = [&](int slot) {
    if (dbg && blockIdx.x == 0) {
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      dbg[slot] = tns;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  using Cfg = TcCfg<BN, A_MN, B_MN, SPLIT, RB>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: [A_hi | B_hi | A_lo | B_lo]  (RB: [A_hi | A_lo], B resident after the stages)
  unsigned char* res = base + kStages * Cfg::STAGE_BYTES;
  auto a_hi = [&](int s) { return base + s * Cfg::STAGE_BYTES; };
  auto a_lo = [&](int s) { return base + s * Cfg::STAGE_BYTES + (RB ? Cfg::A_BYTES : Cfg::A_BYTES + Cfg::B_BYTES); };
  auto b_hi = [&](int s, int kt) {
    return RB ? res + kt * Cfg::NSPLIT * Cfg::B_BYTES : base + s * Cfg::STAGE_BYTES + Cfg::A_BYTES;
  };
  auto b_lo = [&](int s, int kt) {
    return RB ? res + kt * Cfg::NSPLIT * Cfg::B_BYTES + Cfg::B_BYTES
              : base + s * Cfg::STAGE_BYTES + 2 * Cfg::A_BYTES + Cfg::B_BYTES;
  };
  uint64_t* bars = reinterpret_cast<uint64_t*>(res + Cfg::RES_BYTES);
  uint64_t* full = bars;                  // TMA landed
  uint64_t* conv = bars + kStages;        // split done
  uint64_t* empty = bars + 2 * kStages;   // MMA consumed the stage
  uint64_t* accf = bars + 3 * kStages;    // [2] accumulator ready
  uint64_t* acce = bars + 3 * kStages + 2;  // [2] accumulator drained
  uint64_t* bres = bars + 3 * kStages + 4;  // resident B landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kStages + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles = (K + kBK - 1) / kBK;
  const int num_n = (N + BN - 1) / BN, num_m = (M + kBM - 1) / kBM;
  const int total = batches * num_m * num_n;
  auto decode = [&](int t, int& b, int& m0, int& n0) {
    const int nb = t % num_n;
    const int r = t / num_n;
    m0 = (r % num_m) * kBM;
    b = r / num_m;
    n0 = nb * BN;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], SPLIT == 3 ? kConv : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accf[a], 1);
      mbar_init(&acce[a], 128);
    }
    mbar_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: two BN-column fp32 accumulators (128 lanes)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (RB && SPLIT == 3) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
    if (epi_mode == 3) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: everything above overlaps the previous kernel's
  // tail; operands are read (and C written) only after it has completed.  The next
  // kernel in the stream may start its own prologue as SMs free up.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      if constexpr (RB) {  // the constant B (hi and precomputed lo), once per CTA
        mbar_expect_tx(bres, ktiles * Cfg::NSPLIT * Cfg::B_BYTES);
        for (int kt = 0; kt < ktiles; ++kt) {
          tma_load_3d(b_hi(0, kt), &tmB, bres, kt * kBK, 0, 0);
          if (SPLIT == 3) tma_load_3d(b_lo(0, kt), &tmBlo, bres, kt * kBK, 0, 0);
        }
      }
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int b, m0, n0;
        decode(t, b, m0, n0);
        for (int kt = 0; kt < ktiles; ++kt, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          if (it == 0) stamp(2);
          mbar_expect_tx(&full[s], RB ? Cfg::A_BYTES : Cfg::A_BYTES + Cfg::B_BYTES);
          const int k0 = kt * kBK;
          if (!A_MN) {
            tma_load_3d(a_hi(s), &tmA, &full[s], k0, m0, b);
          } else {
            for (int c = 0; c < kBM / 32; ++c) tma_load_3d(a_hi(s) + c * 4096, &tmA, &full[s], m0 + 32 * c, k0, b);
          }
          if constexpr (!RB) {
            if (!B_MN) {
              tma_load_3d(b_hi(s, kt), &tmB, &full[s], k0, n0, b);
            } else {
              for (int c = 0; c < BN / 32; ++c)
                tma_load_3d(b_hi(s, kt) + c * 4096, &tmB, &full[s], n0 + 32 * c, k0, b);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BN, A_MN, B_MN);
    const uint32_t lboA = A_MN ? mn_lbo : 16u, lboB = B_MN ? mn_lbo : 16u;
    const uint32_t sboA = A_MN ? mn_sbo : 1024u, sboB = B_MN ? mn_sbo : 1024u;
    int it = 0, j = 0;
    if (RB) mbar_wait(bres, 0);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++j) {
      const int a = j & 1;
      mbar_wait(&acce[a], ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(a * BN);
      for (int kt = 0; kt < ktiles; ++kt, ++it) {
        const int s = it % kStages;
        mbar_wait(SPLIT == 3 ? &conv[s] : &full[s], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            // K-major: a K=8 step is 32 bytes along the swizzled row; MN-major: eight 128-byte K rows
            const uint32_t koff = (A_MN ? 1024u : 32u) * kk;
            const uint32_t kofb = (B_MN ? 1024u : 32u) * kk;
            const uint64_t dah = umma_desc(smem_u32(a_hi(s)) + koff, lboA, sboA, A_MN);
            const uint64_t dbh = umma_desc(smem_u32(b_hi(s, kt)) + kofb, lboB, sboB, B_MN);
            const uint32_t accum = (kt > 0 || kk > 0) ? 1u : 0u;
            umma_tf32(dacc, dah, dbh, idesc, accum);
            if constexpr (SPLIT == 3) {
              const uint64_t dal = umma_desc(smem_u32(a_lo(s)) + koff, lboA, sboA, A_MN);
              const uint64_t dbl = umma_desc(smem_u32(b_lo(s, kt)) + kofb, lboB, sboB, B_MN);
              umma_tf32(dacc, dah, dbl, idesc, 1u);
              umma_tf32(dacc, dal, dbh, idesc, 1u);
            }
          }
          if (it == 0) stamp(4);
          umma_commit(&empty[s]);  // stage reusable once these MMAs complete
          if (kt == ktiles - 1) umma_commit(&accf[a]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- 3xTF32 split
    if constexpr (SPLIT == 3) {
      const int cv = threadIdx.x - 64;  // 0 .. kConv-1
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        for (int kt = 0; kt < ktiles; ++kt, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          split_tile<Cfg::A_BYTES / 16>(reinterpret_cast<float4*>(a_hi(s)), reinterpret_cast<float4*>(a_lo(s)), cv,
                                        raw_hi);
          if constexpr (!RB)
            split_tile<Cfg::B_BYTES / 16>(reinterpret_cast<float4*>(b_hi(s, kt)),
                                          reinterpret_cast<float4*>(b_lo(s, kt)), cv, raw_hi);
          fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
          if (it == 0 && cv == 0) stamp(3);
          mbar_arrive(&conv[s]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp - 8;  // TMEM lane quarter of this warp (warps 8-11)
    // two 4 KB store boxes per warp (1 KB aligned: 128B-swizzle atoms)
    unsigned char* ebuf = res + Cfg::RES_BYTES + 1024 + q * 2 * 4096;
    int nbox = 0;
    int j = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++j) {
      int b, m0, n0;
      decode(t, b, m0, n0);
      const int a = j & 1;
      mbar_wait(&accf[a], (j >> 1) & 1);
      if (j == 0 && q == 0 && lane == 0) stamp(5);
      tc_fence_after();
      const int row0 = m0 + 32 * q;
      float* cb = C + (int64_t)b * sc;
#pragma unroll 1
      for (int c0 = 0; c0 < BN && n0 + c0 < N; c0 += 32) {
        uint32_t r[32];
        const bool tl = (j == 0 && q == 0 && lane == 0 && c0 < 96);
        if (tl) stamp(8 + 2 * (c0 / 32));
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * BN + c0), r);
        if (tl) stamp(9 + 2 * (c0 / 32));
        if (epi_mode == 3) {
          // registers -> 128B-swizzled smem box (row = lane, 16-byte chunk jj at jj ^ (lane & 7))
          // -> one TMA tensor store per warp; the TMA unit clips rows / columns past M / N
          unsigned char* box = ebuf + (nbox & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();  // the store that last used this box has read it
          __syncwarp();
          if (!ct) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              *reinterpret_cast<float4*>(box + lane * 128 + ((jj ^ (lane & 7)) << 4)) =
                  make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                              __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
          } else {  // C^T: box row = output column, 32 consecutive M-rows (lanes) per box row
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              *reinterpret_cast<float*>(box + jj * 128 + (((lane >> 2) ^ (jj & 7)) << 4) + ((lane & 3) << 2)) =
                  __uint_as_float(r[jj]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0 && row0 < M) {
            if (!ct)
              tma_store_3d(&tmC, box, n0 + c0, row0, b);
            else
              tma_store_3d(&tmC, box, row0, n0 + c0, b);
            bulk_commit();
          }
          ++nbox;
        } else if (epi_mode == 1) {
          // each thread stores its row segment with 16-byte vector stores
          const int row = row0 + lane;
          if (row < M) {
            float* dst = cb + (int64_t)row * ldc + n0 + c0;
            if (n0 + c0 + 32 <= N && (ldc & 3) == 0) {
              float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
                d4[jj] = make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                                     __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (n0 + c0 + jj < N) dst[jj] = __uint_as_float(r[jj]);
            }
          }
        }
      }
      tc_fence_before();
      if (j == 0 && q == 0 && lane == 0) stamp(6);
      mbar_arrive(&acce[a]);  // accumulator a may be overwritten
    }
    if (lane == 0) bulk_wait_all();  // TMA stores complete before the CTA retires
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (lane == 0) stamp(7);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ 3xTF32 with A in TMEM
// The split operands of A never touch shared memory twice: four converter
// warps (one per TMEM lane quarter) read their rows of the raw TMA tile once,
// and write hi = trunc(x) and lo = round(x - hi) straight into tensor memory
// with tcgen05.st; the three MMAs per K=8 step then take A from TMEM
// (tcgen05.mma ... [a_tmem], b_desc), so shared memory carries only the TMA
// writes, one converter read of A, and the B operand reads.  For a K-major A
// the TMA tile keeps the 128B swizzle (conflict-free row reads); an MN-major A
// (slice-major transform input) is fetched unswizzled as [k][32 rows] boxes,
// read down the rows.  B is split in shared memory by two more warps, or is a
// resident constant with a precomputed lo part (RB).
constexpr int kTm3 = 4;                   // TMEM A stages (hi + lo, 64 columns each)
constexpr int kThreads3 = 512;            // 16 warps: TMA, MMA, 4 A converters, 2 B converters, 8 epilogue
// converter threads: warps 2-5 for A; for B warps 6-7 plus, without a resident B (the
// epilogue then has 4 warps), warps 12-15
constexpr int kConvA = 128, kConvB = 192;

template <int BN, bool A_MN, bool B_MN, bool RB>
struct Tc3Cfg {
  static constexpr int A_BYTES = kBM * kBK * 4;  // 16 KB raw A tile
  static constexpr int B_BYTES = BN * kBK * 4;
  static constexpr int STAGE_BYTES = RB ? A_BYTES : A_BYTES + 2 * B_BYTES;  // [A | B_hi | B_lo]
  // shared-memory ring: with a resident B a stage holds only the raw A tile and is
  // released as soon as the converters have read it, so a deeper ring keeps more
  // HBM reads in flight; otherwise B lives in the stage until its MMAs complete
  static constexpr int SMS = RB ? 5 : 4;
  static constexpr int RES_BYTES = RB ? kRbMaxKt * 2 * B_BYTES : 0;
  // epilogue warps: 8 (two per TMEM lane quarter, alternate 32-column chunks) with a
  // resident B; 4 otherwise (shared memory is taken by the B stages)
  static constexpr int EPW = RB ? 8 : 4;
  static constexpr int EPI_BYTES = EPW * 2 * 4096;
  static constexpr int SMEM = SMS * STAGE_BYTES + RES_BYTES + 1024 + 1024 + EPI_BYTES;
  static constexpr int ACOL = 2 * BN;  // TMEM column of the first A stage (after two accumulators)
  static_assert(ACOL + kTm3 * 64 <= 512, "accumulators + A stages must fit in TMEM");
  static_assert(RB || SMS == kTm3, "without a resident B the shared-memory and TMEM rings advance together");
  static_assert(B_BYTES % 1024 == 0 && STAGE_BYTES % 1024 == 0, "1 KB swizzle-atom alignment");
  static_assert(!RB || !B_MN, "resident B is K-major");
};

__device__ __forceinline__ void umma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// warp-uniform issue: every lane executes the call, one elected lane issues the
// instruction, so the operands stay in uniform registers (no per-MMA R2UR
// waterfall, which a lane-0-only branch forces and which halves the MMA rate)
__device__ __forceinline__ void umma_tf32_ta_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// warp-uniform issue with A from shared memory (descriptor), as umma_tf32_ta_w
__device__ __forceinline__ void umma_tf32_w(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// optional per-batch extras (the SVT recomposition, ltb_svd.cu): K limited to the
// kept count (a tile with no K blocks stores zeros), output rows / columns scaled
struct Tc3Extras {
  const int* klim;       // batch, or null
  const float* rscale;   // batch x M, or null
  const float* cscale;   // batch x N, or null
  const int* skip;       // device flag, or null
  float* c_direct;       // C^T output written with coalesced per-column stores (lanes = rows), or null
  int64_t ldc, sc;
  // C written by the warps themselves (each 32 x 32 box staged in shared memory, then read
  // back four 128-byte rows per instruction and stored coalesced) instead of TMA stores:
  // keeps the epilogue out of the TMA unit's queue, which the operand loads fill; or null
  float* c_lsu;
  int c_vec;  // C, ldc and sc allow 16-byte vector stores
};

template <int BN, bool A_MN, bool B_MN, bool RB>
__global__ void __launch_bounds__(kThreads3, 1)
    tc3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmC, int M, int N,
               int K, int batches, uint32_t mn_lbo, uint32_t mn_sbo, int ct, Tc3Extras ex,
               unsigned long long* dbg) {
  using Cfg = Tc3Cfg<BN, A_MN, B_MN, RB>;
  // optional timeline (CTA 0, %globaltimer ns): same slots as tc_gemm_tf32_kernel
  auto stamp = [&](int slot) {
    if (dbg && blockIdx.x == 0) {
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      dbg[slot] = tns;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  auto cta_stamp = [&](int k) {  // per-CTA start / end (slots 256 + 2 * CTA + k)
    if (dbg) {
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      dbg[256 + 2 * blockIdx.x + k] = tns;
    }
  };
  if (threadIdx.x == 0) cta_stamp(0);
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SMS = Cfg::SMS;
  unsigned char* res = base + SMS * Cfg::STAGE_BYTES;
  auto a_raw = [&](int s) { return base + s * Cfg::STAGE_BYTES; };
  auto b_hi = [&](int s, int kt) {
    return RB ? res + kt * 2 * Cfg::B_BYTES : base + s * Cfg::STAGE_BYTES + Cfg::A_BYTES;
  };
  auto b_lo = [&](int s, int kt) {
    return RB ? res + kt * 2 * Cfg::B_BYTES + Cfg::B_BYTES : base + s * Cfg::STAGE_BYTES + Cfg::A_BYTES + Cfg::B_BYTES;
  };
  uint64_t* bars = reinterpret_cast<uint64_t*>(res + Cfg::RES_BYTES);
  uint64_t* full = bars;                  // [SMS] TMA landed
  uint64_t* sfree = bars + SMS;           // [SMS] smem stage reusable
  uint64_t* tfull = bars + 2 * SMS;       // [kTm3] A in TMEM (and B split) for the k-block
  uint64_t* tfree = tfull + kTm3;         // [kTm3] MMAs reading the TMEM stage completed
  uint64_t* accf = tfree + kTm3;          // [2] accumulator ready
  uint64_t* acce = accf + 2;              // [2] accumulator drained
  uint64_t* bres = acce + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles = (K + kBK - 1) / kBK;
  const int num_n = (N + BN - 1) / BN, num_m = (M + kBM - 1) / kBM;
  int total = batches * num_m * num_n;
  auto decode = [&](int t, int& b, int& m0, int& n0) {
    const int nb = t % num_n;
    const int r = t / num_n;
    m0 = (r % num_m) * kBM;
    b = r / num_m;
    n0 = nb * BN;
  };
  auto ktiles_of = [&](int b) {  // K blocks of batch b (all of them without a limit)
    if (!ex.klim) return ktiles;
    const int kb = min(K, max(ex.klim[b], 0));
    return (kb + kBK - 1) / kBK;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < SMS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], RB ? kConvA : 1);
    }
    for (int s = 0; s < kTm3; ++s) {
      mbar_init(&tfull[s], kConvA + (RB ? 0 : kConvB));
      mbar_init(&tfree[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accf[a], 1);
      mbar_init(&acce[a], 32 * Cfg::EPW);
    }
    mbar_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (RB) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) stamp(1);
  // device-side stop flag (PGA), read after the dependency wait: no tiles at all
  if (ex.skip && *ex.skip) total = 0;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      if (RB && total > 0) {
        mbar_expect_tx(bres, ktiles * 2 * Cfg::B_BYTES);
        for (int kt = 0; kt < ktiles; ++kt) {
          tma_load_3d(b_hi(0, kt), &tmB, bres, kt * kBK, 0, 0);
          tma_load_3d(b_lo(0, kt), &tmBlo, bres, kt * kBK, 0, 0);
        }
      }
      int it = 0, j_t = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++j_t) {
        int b, m0, n0;
        decode(t, b, m0, n0);
        const int kt_b = ktiles_of(b);
        for (int kt = 0; kt < kt_b; ++kt, ++it) {
          const int s = it % SMS;
          mbar_wait(&sfree[s], ((it / SMS) & 1) ^ 1);
          if (it == 0) stamp(2);
          if (kt == 0 && j_t < 16) stamp(16 + j_t);
          mbar_expect_tx(&full[s], RB ? Cfg::A_BYTES : Cfg::A_BYTES + Cfg::B_BYTES);
          const int k0 = kt * kBK;
          if (!A_MN) {
            tma_load_3d(a_raw(s), &tmA, &full[s], k0, m0, b);
          } else {
            for (int c = 0; c < kBM / 32; ++c) tma_load_3d(a_raw(s) + c * 4096, &tmA, &full[s], m0 + 32 * c, k0, b);
          }
          if constexpr (!RB) {
            if (!B_MN) {
              tma_load_3d(b_hi(s, kt), &tmB, &full[s], k0, n0, b);
            } else {
              for (int c = 0; c < BN / 32; ++c)
                tma_load_3d(b_hi(s, kt) + c * 4096, &tmB, &full[s], n0 + 32 * c, k0, b);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BN, false, B_MN);
    const uint32_t lboB = B_MN ? mn_lbo : 16u, sboB = B_MN ? mn_sbo : 1024u;
    int it = 0, j = 0;
    if (RB && total > 0) mbar_wait(bres, 0);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++j) {
      const int a = j & 1;
      int b, m0, n0;
      decode(t, b, m0, n0);
      const int kt_b = ktiles_of(b);
      mbar_wait(&acce[a], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(a * BN);
      if (kt_b == 0) {  // nothing to accumulate: the epilogue stores zeros
        if (lane == 0) mbar_arrive(&accf[a]);
        __syncwarp();
        continue;
      }
      for (int kt = 0; kt < kt_b; ++kt, ++it) {
        const int s = it % SMS, ts = it % kTm3;
        mbar_wait(&tfull[ts], (it / kTm3) & 1);
        tc_fence_after();
        if (lane == 0 && it < 16) stamp(80 + it);
        const uint32_t ahi = tmem + (uint32_t)(Cfg::ACOL + 64 * ts), alo = ahi + 32;
        // descriptor address field = byte address >> 4 (< 2^14 for any shared-memory
        // address), so the K step is added to the descriptor directly
        const uint64_t dbh0 = umma_desc(smem_u32(b_hi(s, kt)), lboB, sboB, B_MN);
        const uint64_t dbl0 = umma_desc(smem_u32(b_lo(s, kt)), lboB, sboB, B_MN);
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint64_t kof = (uint64_t)(((B_MN ? 1024u : 32u) * kk) >> 4);
          umma_tf32_ta_w(dacc, ahi + 8 * kk, dbh0 + kof, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
          umma_tf32_ta_w(dacc, ahi + 8 * kk, dbl0 + kof, idesc, 1u);
          umma_tf32_ta_w(dacc, alo + 8 * kk, dbh0 + kof, idesc, 1u);
        }
        if (lane == 0) {
          if (it == 0) stamp(4);
          if (it < 16) stamp(112 + it);
          if (kt == kt_b - 1 && j < 16) stamp(32 + j);
        }
        umma_commit_w(&tfree[ts]);
        if (!RB) umma_commit_w(&sfree[s]);  // B of this smem stage has been read
        if (kt == kt_b - 1) umma_commit_w(&accf[a]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------------------------------------------------------- A -> TMEM (hi, lo)
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int row = 32 * q + lane;   // tile row of this thread
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int b, m0, n0;
      decode(t, b, m0, n0);
      const int kt_b = ktiles_of(b);
      for (int kt = 0; kt < kt_b; ++kt, ++it) {
        const int s = it % SMS, ts = it % kTm3;
        mbar_wait(&full[s], (it / SMS) & 1);
        if (threadIdx.x == 64 && it < 16) stamp(96 + it);
        uint32_t hi[32], lo[32];
        const unsigned char* ab = a_raw(s);
        if (!A_MN) {  // 128B-swizzled rows: 16-byte chunk c of row r sits at c ^ (r & 7)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(ab + row * 128 + ((c ^ (row & 7)) << 4));
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float h = tf32_trunc(x[e]);
              hi[4 * c + e] = __float_as_uint(h);
              lo[4 * c + e] = __float_as_uint(tf32_round(x[e] - h));
            }
          }
        } else {  // unswizzled [k][32 rows] boxes, one per 32-row chunk
          const float* cb = reinterpret_cast<const float*>(ab + (row >> 5) * 4096) + (row & 31);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = cb[32 * k];
            const float h = tf32_trunc(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(tf32_round(x - h));
          }
        }
        if (RB) mbar_arrive(&sfree[s]);  // the raw tile is in registers: the TMA may refill the stage
        mbar_wait(&tfree[ts], ((it / kTm3) & 1) ^ 1);  // MMAs of the TMEM stage's previous k-block done
        tc_fence_after();
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(Cfg::ACOL + 64 * ts);
        tmem_st32(tq, hi);
        tmem_st32(tq + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        if (it == 0 && threadIdx.x == 64) stamp(3);
        if (threadIdx.x == 64 && it < 16) stamp(64 + it);
        if (threadIdx.x == 160 && it < 16) stamp(128 + it);
        mbar_arrive(&tfull[ts]);
      }
    }
  } else if (warp < 8 || (!RB && warp >= 12)) {
    // ---------------------------------------------------------------- B split in shared memory
    if constexpr (!RB) {
      const int cv = warp < 8 ? threadIdx.x - 192 : threadIdx.x - 320;  // 0 .. kConvB-1
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int b, m0, n0;
        decode(t, b, m0, n0);
        const int kt_b = ktiles_of(b);
        for (int kt = 0; kt < kt_b; ++kt, ++it) {
          const int s = it % SMS;
          mbar_wait(&full[s], (it / SMS) & 1);
          float4* bh = reinterpret_cast<float4*>(b_hi(s, kt));
          float4* bl = reinterpret_cast<float4*>(b_lo(s, kt));
#pragma unroll 4
          for (int i = cv; i < Cfg::B_BYTES / 16; i += kConvB) {
            const float4 x = bh[i];
            const float4 h = make_float4(tf32_trunc(x.x), tf32_trunc(x.y), tf32_trunc(x.z), tf32_trunc(x.w));
            bl[i] = make_float4(tf32_round(x.x - h.x), tf32_round(x.y - h.y), tf32_round(x.z - h.z),
                                tf32_round(x.w - h.w));
          }
          fence_proxy_async();
          mbar_arrive(&tfull[s]);  // SMS == kTm3 here
        }
      }
    }
  } else if (warp < 8 + Cfg::EPW) {
    // ---------------------------------------------------------------- epilogue (TMA tensor stores)
    const int q = warp & 3;                         // TMEM lane quarter
    const int half = (warp - 8) >> 2;               // chunk parity (EPW == 8) or 0
    constexpr int CSTEP = 32 * (Cfg::EPW / 4);      // column stride between this warp's chunks
    unsigned char* ebuf = res + Cfg::RES_BYTES + 1024 + (warp - 8) * 2 * 4096;
    int nbox = 0, j = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++j) {
      int b, m0, n0;
      decode(t, b, m0, n0);
      const int a = j & 1;
      mbar_wait(&accf[a], (j >> 1) & 1);
      if (j == 0 && q == 0 && lane == 0) stamp(5);
      const bool tl = (j < 4 && warp == 8 && lane == 0);
      int ck = 0;
      if (tl) stamp(160 + 4 * j);
      tc_fence_after();
      const int row0 = m0 + 32 * q;
      const bool zero = ktiles_of(b) == 0;
      const float rs = (ex.rscale && row0 + lane < M) ? ex.rscale[(int64_t)b * M + row0 + lane] : 1.f;
#pragma unroll 1
      for (int c0 = 32 * half; c0 < BN && n0 + c0 < N; c0 += CSTEP) {
        uint32_t r[32];
        if (!zero) {
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * BN + c0), r);
          if (tl && ck < 2) stamp(179 + 8 * j + 4 * ck);
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) r[jj] = 0u;
        }
        if (ex.rscale || ex.cscale) {
          const float* cs = ex.cscale ? ex.cscale + (int64_t)b * N + n0 + c0 : nullptr;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const float c = (cs && n0 + c0 + jj < N) ? cs[jj] : 1.f;
            r[jj] = __float_as_uint(__uint_as_float(r[jj]) * rs * c);
          }
        }
        if (ct && ex.c_direct) {
          // C^T: for each output column the 32 lanes hold 32 consecutive rows -> one 128-byte store
          const int row = row0 + lane;
          if (row < M) {
            float* cb = ex.c_direct + (int64_t)b * ex.sc + row;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (n0 + c0 + jj < N) cb[(int64_t)(n0 + c0 + jj) * ex.ldc] = __uint_as_float(r[jj]);
          }
          continue;
        }
        unsigned char* box = ebuf + (nbox & 1) * 4096;
        if (!ex.c_lsu && lane == 0) bulk_wait_read<1>();
        __syncwarp();
        if (tl && ck < 2) stamp(176 + 8 * j + 4 * ck);
        if (!ct) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            *reinterpret_cast<float4*>(box + lane * 128 + ((jj ^ (lane & 7)) << 4)) =
                make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                            __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            *reinterpret_cast<float*>(box + jj * 128 + (((lane >> 2) ^ (jj & 7)) << 4) + ((lane & 3) << 2)) =
                __uint_as_float(r[jj]);
        }
        if (tl && ck < 2) stamp(177 + 8 * j + 4 * ck);
        if (ex.c_lsu) {
          // box row r (output row of C, or of C^T when ct), 16-byte chunk cc at
          // r * 128 + ((cc ^ (r & 7)) << 4): 8 lanes per row, 4 rows per instruction
          __syncwarp();
          const int r_lim = ct ? N : M, c_lim = ct ? M : N;
          const int gr0 = ct ? n0 + c0 : row0, gc = (ct ? row0 : n0 + c0) + 4 * (lane & 7);
          float* cbase = ex.c_lsu + (int64_t)b * ex.sc;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3), gr = gr0 + r;
            const float4 v = *reinterpret_cast<const float4*>(box + r * 128 + (((lane & 7) ^ (r & 7)) << 4));
            if (gr < r_lim) {
              float* dst = cbase + (int64_t)gr * ex.ldc + gc;
              if (ex.c_vec && gc + 3 < c_lim) {
                *reinterpret_cast<float4*>(dst) = v;
              } else {
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (gc + u < c_lim) dst[u] = e[u];
              }
            }
          }
          __syncwarp();
          if (tl && ck < 2) stamp(162 + 4 * j + ck);
          ++ck;
          ++nbox;
          continue;
        }
        fence_proxy_async();
        if (tl && ck < 2) stamp(178 + 8 * j + 4 * ck);
        __syncwarp();
        if (lane == 0 && row0 < M) {
          if (!ct)
            tma_store_3d(&tmC, box, n0 + c0, row0, b);
          else
            tma_store_3d(&tmC, box, row0, n0 + c0, b);
          bulk_commit();
          if (tl) stamp(162 + 4 * j + min(ck, 1));
          ++ck;
        }
        ++nbox;
      }
      tc_fence_before();
      if (j == 0 && q == 0 && lane == 0) stamp(6);
      if (j < 16 && q == 0 && half == 0 && lane == 0) stamp(48 + j);
      mbar_arrive(&acce[a]);
    }
    if (!ex.c_lsu && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (lane == 0) stamp(7);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (lane == 0) cta_stamp(1);
  }
}

// ------------------------------------------------------------------ host: tensor maps
// MN-major 128B-swizzle descriptor strides (bytes): LBO = MN-chunk stride, SBO = 8-row K-group stride
constexpr uint32_t g_mn_lbo = 4096, g_mn_sbo = 512;
// 1: leave the fp32 tile in place as the "hi" operand (valid iff the tensor core
// truncates fp32 -> tf32); 0: store hi = x with the low 13 bits cleared
constexpr int g_raw_hi = 1;
// epilogue store mode: 3 swizzled smem boxes + TMA tensor stores (default, needs a
// C tensor map), 1 direct per-thread row stores, 2 no stores (diagnostic only)
constexpr int g_epi_mode = 3;
// programmatic dependent launch on (1) / off (0)
constexpr int g_pdl = 1;
// resident constant-B variant allowed (1) / off (0)
constexpr int g_rb = 1;
// 3xTF32 with A staged in TMEM (tc3_kernel) (1) / split in shared memory (0)
constexpr int g_tc3 = 1;
// transposed outputs: coalesced direct stores (1) / smem box + TMA store (0)
constexpr int g_ct_direct = 0;
// tc3 epilogue: warp-coalesced stores from the shared-memory box (1) / TMA tensor stores (0,
// measured faster on the config-2 step: 51 vs 63 us)
constexpr int g_epi_lsu = 0;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  }
  return fn;
}

// 3D fp32 map: dims {inner, rows, batch}, box {32, box_rows, 1}, 128B swizzle, zero OOB fill
// small cache of encoded tensor maps: the encode call costs microseconds of
// host time, and repeated calls on the same buffers (benchmark steps, PGA
// iterations) reuse identical maps
struct MapKey {
  const float* ptr;
  int64_t inner, rows, batch, ld, bstride;
  int box_rows;
  int swz;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && rows == o.rows && batch == o.batch && ld == o.ld &&
           bstride == o.bstride && box_rows == o.box_rows && swz == o.swz;
  }
};
struct MapEntry {
  MapKey key;
  CUtensorMap map;
  bool valid;
};
MapEntry g_map_cache[32];
int g_map_next = 0;

bool make_map(CUtensorMap* map, const float* ptr, int64_t inner, int64_t rows, int64_t batch, int64_t ld,
              int64_t bstride, int box_rows, int swz = 0) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 4) % 16 || (bstride * 4) % 16) return false;
  const MapKey key{ptr, inner, rows, batch, ld, bstride, box_rows, swz};
  for (auto& e : g_map_cache)
    if (e.valid && e.key == key) {
      *map = e.map;
      return true;
    }
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(bstride * 4)};
  cuuint32_t box[3] = {32u, (cuuint32_t)box_rows, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  const bool ok = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz == 1   ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                      : swz == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                 : CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  if (ok) {
    MapEntry& e = g_map_cache[g_map_next];
    g_map_next = (g_map_next + 1) % 32;
    e.key = key;
    e.map = *map;
    e.valid = true;
  }
  return ok;
}

template <int BN, bool A_MN, bool B_MN, int SPLIT, bool RB>
int launch_tc(ltb_ctx* ctx, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mblo,
              const CUtensorMap& mc, bool have_mc, int ct, float* C, int64_t ldc, int64_t sc, int64_t batch, int M,
              int N, int K) {
  using Cfg = TcCfg<BN, A_MN, B_MN, SPLIT, RB>;
  const uint32_t mn_lbo = g_mn_lbo, mn_sbo = g_mn_sbo;
  auto kern = tc_gemm_tf32_kernel<BN, A_MN, B_MN, SPLIT, RB>;
  LTB_TRY(ensure_smem(ctx, kern, Cfg::SMEM));
  // persistent: one CTA per SM, tiles strided over the grid
  const int64_t tiles = batch * (int64_t)((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int grid = (int)std::min<int64_t>(tiles, ctx->num_sms);
  const int epi = (g_epi_mode == 3 && !have_mc) ? 1 : g_epi_mode;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LTB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, ma, mb, mblo, mc, C, ldc, sc, M, N, K, (int)batch, mn_lbo, mn_sbo,
                                       g_raw_hi, ctx->opt_tc_timeline, epi, ct));
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

template <int BN, bool A_MN, bool B_MN, bool RB>
int launch_tc3(ltb_ctx* ctx, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mblo,
               const CUtensorMap& mc, int ct, int64_t batch, int M, int N, int K, const Tc3Extras& ex) {
  using Cfg = Tc3Cfg<BN, A_MN, B_MN, RB>;
  auto kern = tc3_kernel<BN, A_MN, B_MN, RB>;
  LTB_TRY(ensure_smem(ctx, kern, Cfg::SMEM));
  const int64_t tiles = batch * (int64_t)((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int grid = (int)std::min<int64_t>(tiles, ctx->num_sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads3);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LTB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, ma, mb, mblo, mc, M, N, K, (int)batch, g_mn_lbo, g_mn_sbo, ct, ex,
                                       ctx->opt_tc_timeline));
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

}  // namespace

// C[b] = op(A[b]) op(B[b]) in fp32 on tcgen05 (3xTF32 when split == 3).
// a_mn: A stored K x M (else M x K); b_mn: B stored K x N (else N x K).
// c_trans: write C^T (C stored N x M with leading dimension ldc) instead of C.
// b_lo: optional precomputed lo part of a constant K-major B (batch 1): with
// N <= 96 and K <= 128 B then stays resident in shared memory for the whole
// launch (the transform's Kronecker matrix) and only A is split on the fly.
// Returns LTB_EUNSUPPORTED (no error text) when the shape / alignment / driver
// cannot use the tensor-core path; the caller then falls back.
int ltb_tc_gemm_f32(ltb_ctx* ctx, int64_t batch, int64_t M, int64_t N, int64_t K, bool a_mn, const float* A,
                    int64_t lda, int64_t sa, bool b_mn, const float* B, int64_t ldb, int64_t sb, float* C,
                    int64_t ldc, int64_t sc, int split, bool c_trans, const float* b_lo, const int* klim,
                    const float* rscale, const float* cscale, const int* skip) {
  const bool c_vec = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && ldc % 4 == 0 && (batch == 1 || sc % 4 == 0);
  const Tc3Extras ex{klim, rscale, cscale, skip, (c_trans && g_ct_direct) ? C : nullptr, ldc, sc,
                     g_epi_lsu ? C : nullptr, c_vec ? 1 : 0};
  const bool extras = klim || rscale || cscale || skip;
  if (batch < 1 || M < 1 || N < 1 || K < 1 || batch > 65535) return LTB_EUNSUPPORTED;
  if (M > (1 << 30) || N > (1 << 30) || K > (1 << 30)) return LTB_EUNSUPPORTED;
  if ((M + kBM - 1) / kBM > 65535) return LTB_EUNSUPPORTED;
  const bool rb = b_lo && g_rb && split == 3 && !b_mn && (batch == 1 || sb == 0) && N <= 96 &&
                  K <= kRbMaxKt * kBK;
  const int BN = rb ? 96 : 128;
  CUtensorMap ma, mb, mblo;
  // A: K-major -> dims {K, M}, box {32, 128};  MN-major -> dims {M, K}, box {32 (M), 32 (K)}
  const bool okA = a_mn ? make_map(&ma, A, M, K, batch, lda, sa, kBK, true) : make_map(&ma, A, K, M, batch, lda, sa, kBM);
  const bool okB = b_mn ? make_map(&mb, B, N, K, batch, ldb, sb, kBK, true) : make_map(&mb, B, K, N, batch, ldb, sb, BN);
  const bool okBlo = rb ? make_map(&mblo, b_lo, K, N, 1, ldb, 0, BN) : true;
  if (!rb) std::memset(&mblo, 0, sizeof(mblo));
  if (!okA || !okB || !okBlo) return LTB_EUNSUPPORTED;
  // C: dims {N, M, batch} (C^T: {M, N, batch}), box {32, 32, 1}, 128B swizzle (TMA-store epilogue)
  CUtensorMap mc;
  const bool okC = c_trans ? make_map(&mc, C, M, N, batch, ldc, sc, 32) : make_map(&mc, C, N, M, batch, ldc, sc, 32);
  if (!okC) {
    if (c_trans) return LTB_EUNSUPPORTED;  // the transposed store needs the TMA epilogue
    std::memset(&mc, 0, sizeof(mc));
  }
  const int m = (int)M, n = (int)N, k = (int)K, ct = c_trans ? 1 : 0;
  if (extras && !(split == 3 && g_tc3 && okC)) return LTB_EUNSUPPORTED;  // extras live in tc3_kernel only
  if (split == 3 && g_tc3 && okC) {
    // A staged in TMEM (tc3_kernel): an MN-major A is fetched unswizzled
    CUtensorMap ma3;
    const bool ok3 = a_mn ? make_map(&ma3, A, M, K, batch, lda, sa, kBK, 2) : (ma3 = ma, true);
    if (ok3) {
#define LTB_TC3(BNv, AM, BM_, RBv) launch_tc3<BNv, AM, BM_, RBv>(ctx, ma3, mb, mblo, mc, ct, batch, m, n, k, ex)
      if (rb) return a_mn ? LTB_TC3(96, true, false, true) : LTB_TC3(96, false, false, true);
      if (!a_mn && !b_mn) return LTB_TC3(128, false, false, false);
      if (!a_mn && b_mn) return LTB_TC3(128, false, true, false);
      if (a_mn && !b_mn) return LTB_TC3(128, true, false, false);
      return LTB_TC3(128, true, true, false);
#undef LTB_TC3
    }
  }
#define LTB_TC(BNv, AM, BM_, SP, RBv) \
  launch_tc<BNv, AM, BM_, SP, RBv>(ctx, ma, mb, mblo, mc, okC, ct, C, ldc, sc, batch, m, n, k)
  if (rb) return a_mn ? LTB_TC(96, true, false, 3, true) : LTB_TC(96, false, false, 3, true);
  if (split == 3) {
    if (!a_mn && !b_mn) return LTB_TC(128, false, false, 3, false);
    if (!a_mn && b_mn) return LTB_TC(128, false, true, 3, false);
    if (a_mn && !b_mn) return LTB_TC(128, true, false, 3, false);
    return LTB_TC(128, true, true, 3, false);
  }
  if (!a_mn && !b_mn) return LTB_TC(128, false, false, 1, false);
  if (!a_mn && b_mn) return LTB_TC(128, false, true, 1, false);
  if (a_mn && !b_mn) return LTB_TC(128, true, false, 1, false);
  return LTB_TC(128, true, true, 1, false);
#undef LTB_TC
}



// test hook: exported C entry for the kernel-level tests (fp32 only)
extern "C" int ltb_tc_gemm(ltb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t k, int a_mn, const void* d_a,
                           int64_t lda, int64_t sa, int b_mn, const void* d_b, int64_t ldb, int64_t sb, void* d_c,
                           int64_t ldc, int64_t sc, int split) {
  int st = ltb_tc_gemm_f32(ctx, batch, m, n, k, a_mn != 0, (const float*)d_a, lda, sa, b_mn != 0, (const float*)d_b,
                           ldb, sb, (float*)d_c, ldc, sc, split, false, nullptr);
  if (st == LTB_EUNSUPPORTED) return ltb_set_error(ctx, LTB_EUNSUPPORTED, "tc_gemm: shape/alignment unsupported");
  return st;
}

// ------------------------------------------------------------------ debug: raw MMA issue rate
// One CTA issues `iters` x 12 kind::tf32 MMAs (M = 128, N = BN, K = 8 each) into one
// accumulator; returns SM cycles from the first issue to the commit's arrival.
// pattern 0: A from shared memory, one A / one B tile; 1: A from TMEM, one A / one B;
// 2: the 3xTF32 order of tc3_kernel (A hi/lo in TMEM, B hi/lo in smem, per K step
// hi*hi, hi*lo, lo*hi); 3: the same MMAs grouped by operand pair (4 x hi*hi, 4 x hi*lo,
// 4 x lo*hi).  pattern | 4: warps 4-7 load TMEM (32 columns each, like the epilogue)
// while the MMAs run; | 8: warps 8-11 store TMEM (like the converters); | 16: warps
// 12-15 stream shared memory (float4 reads + writes); | 32: A at TMEM column 192 (as
// tc3_kernel with BN = 96); | 64: 148 CTAs (one per SM) instead of one; | 128: random
// operand values instead of zeros; | 256: B cycles through 3 K blocks (timing only).
template <int BN>
__global__ void mma_rate_kernel(int pattern, int iters, unsigned long long* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  __shared__ volatile int done;
  constexpr int ABYTES = kBM * 128, BBYTES = BN * 128;
  if (threadIdx.x == 0) done = 0;
  const bool rnd = pattern & 128;
  auto hv = [&](uint32_t i) {  // deterministic pseudo-random value in [-1, 1)
    i = i * 2654435761u + 12345u;
    i ^= i >> 13;
    i *= 0x5bd1e995u;
    i ^= i >> 15;
    return rnd ? (float)(i & 0xFFFFFF) / 8388608.f - 1.f : 0.f;
  };
  for (int i = threadIdx.x; i < (ABYTES + 6 * BBYTES + 32768) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(base)[i] = make_float4(hv(4 * i), hv(4 * i + 1), hv(4 * i + 2), hv(4 * i + 3));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int warp = threadIdx.x >> 5;
  const int mode = pattern & 3;
  if (warp < 4) {  // A hi / lo tiles in TMEM (columns 192 .. 319)
    uint32_t r[32];
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(hv(threadIdx.x * 131 + c * 32 + i + 7777));
      tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 192u + 32u * c, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp >= 4 && warp < 8 && (pattern & 4)) {
    uint32_t r[32];
    unsigned acc = 0;
    while (!done) {
      tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 320u, r);
      acc += r[0];
    }
    if (acc == 12345u) out[1] = acc;
  } else if (warp >= 8 && warp < 12 && (pattern & 8)) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = 0u;
    while (!done) {
      tmem_st32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 416u, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else if (warp >= 12 && (pattern & 16)) {
    float4* sp = reinterpret_cast<float4*>(base + ABYTES + 6 * BBYTES);
    const int t = threadIdx.x - 384;
    while (!done) {
#pragma unroll 4
      for (int i = t; i < 2048; i += 128) {
        float4 v = sp[i];
        v.x += 1.f;
        sp[(i + 64) & 2047] = v;
      }
    }
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_tf32(BN, false, false);
    const uint32_t sa = smem_u32(base), sbh = smem_u32(base + ABYTES), sbl = sbh + BBYTES;
    const uint32_t acol = (pattern & 32) ? 192u : 256u;
    const uint32_t ahi = tmem + acol, alo = tmem + acol + 32u;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_tf32(tmem, umma_desc(sa + 32u * kk, 16u, 1024u), umma_desc(sbh + 32u * kk, 16u, 1024u), idesc,
                      (i | r | kk) ? 1u : 0u);
      } else if (mode == 1) {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_tf32_ta(tmem, ahi + 8u * kk, umma_desc(sbh + 32u * kk, 16u, 1024u), idesc, (i | r | kk) ? 1u : 0u);
      } else if (mode == 2) {
        // | 256: B cycles through 3 K blocks (hi + lo each), like the resident Kronecker matrix
        const uint32_t boff = (pattern & 256) ? (uint32_t)(i % 3) * 2u * BBYTES : 0u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t dbh = umma_desc(sbh + boff + 32u * kk, 16u, 1024u),
                         dbl = umma_desc(sbh + boff + BBYTES + 32u * kk, 16u, 1024u);
          umma_tf32_ta(tmem, ahi + 8u * kk, dbh, idesc, (i | kk) ? 1u : 0u);
          umma_tf32_ta(tmem, ahi + 8u * kk, dbl, idesc, 1u);
          umma_tf32_ta(tmem, alo + 8u * kk, dbh, idesc, 1u);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_tf32_ta(tmem, ahi + 8u * kk, umma_desc(sbh + 32u * kk, 16u, 1024u), idesc, (i | kk) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_tf32_ta(tmem, ahi + 8u * kk, umma_desc(sbl + 32u * kk, 16u, 1024u), idesc, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_tf32_ta(tmem, alo + 8u * kk, umma_desc(sbh + 32u * kk, 16u, 1024u), idesc, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = (unsigned long long)(clock64() - t0);
    done = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int BN>
static int run_mma_rate(int pattern, int iters, unsigned long long* d_out) {
  auto k = mma_rate_kernel<BN>;
  const int smem = kBM * 128 + 6 * BN * 128 + 32768 + 1024;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return LTB_ECUDA;
  k<<<(pattern & 64) ? 148 : 1, 512, smem>>>(pattern, iters, d_out);
  return cudaGetLastError() == cudaSuccess ? LTB_OK : LTB_ECUDA;
}

extern "C" int ltb_tc_debug_mma_rate(int bn, int pattern, int iters, unsigned long long* d_out) {
  switch (bn) {
    case 64: return run_mma_rate<64>(pattern, iters, d_out);
    case 96: return run_mma_rate<96>(pattern, iters, d_out);
    case 128: return run_mma_rate<128>(pattern, iters, d_out);
    case 256: return run_mma_rate<256>(pattern, iters, d_out);
    default: return LTB_EPARAM;
  }
}

// the fused one-launch *_L product (shares this file's helpers)
#include "ltb_lprod_fused.cuh"
