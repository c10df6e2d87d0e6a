// The whole fp32 *_L product (linalg.py:34-43) as ONE persistent tcgen05 kernel.
//
// Included at the end of ltb_tc_gemm.cu: it reuses that file's PTX helpers (TMA, mbarrier,
// tcgen05 MMA / ld / st, the 3xTF32 split, the tensor-map cache).
//
// The three-launch path (K1(A,B) -> K2 -> K1') pays, per launch, the prologue (TMEM
// alloc, barrier init, resident Kronecker load), the pipeline fill (~2.8 us to the first
// landed k-block) and drain (~2 us for the last epilogue), plus a 4-vs-3 tile tail: about
// 8 us of streaming inside ~16 us per phase (profiles/r01_tc3_tile_timeline.txt).  Here
// every CTA (one per SM) runs a loop over ONE ordered list of tiles of all three phases,
// claimed dynamically from a global counter:
//
//   F  forward transforms   D(128 tubes x P) = X K^T, tubes of A then B, transposed store
//                           into the slice-major stacks A-hat, B-hat     (BN = 96, K = P)
//   G  slice GEMMs          C-hat_q = A-hat_q B-hat_q, 128 x 128 tiles     (BN = 128, K = L)
//   I  inverse transforms   D(128 tubes x P) = C-hat^T Kinv^T -> C         (BN = 96, K = P)
//
// A tile may only start once the tiles it reads are complete, so the list is ordered by
// dependency and the dependencies are counted per group, not per phase:
//   F: [A rows 0..127 | all of B | A rows 128..255 | ...]   G: m-block 0, 1, ...   I: row block 0, 1, ...
//   G tiles of m-block b need F group 0 (A rows block 0 and all of B) and F group b;
//   I tiles of row block b need the G tiles of m-block b.
// Each epilogue warp adds its completed tiles to the group's counter (red.release.gpu, after
// waiting for its TMA stores; deferred to the warp's first tile of another group, so a warp
// waits for its stores once per group, not per tile); a producer whose next tile depends on
// an incomplete group spins on ld.acquire.gpu.  Tiles are claimed in list order, so every dependency is held by
// a running CTA: no deadlock, and a CTA that waits does so while other CTAs stream the
// tail of the previous group -- the phases overlap instead of draining at kernel borders.
//
// Per CTA (16 warps): warp 0 TMA producer + tile claimer (publishes tile ids through a
// 4-slot shared-memory queue), warp 1 MMA issuer, warps 2-5 A -> TMEM converters (hi / lo),
// warps 6-7 B-hat converters (G tiles: lo split in shared memory), warps 8-15 epilogue.
// Shared memory: one 152 KB region used either as [resident K or Kinv (hi|lo, 72 KB) |
// 5 x 16 KB raw-A ring] for F / I tiles, or as a 3 x 48 KB [A | B hi | B lo] ring for G
// tiles; when a CTA switches between the two uses the producer first waits for every MMA
// it has issued to complete (each CTA switches at most three times).
namespace {

constexpr int kLpThreads = 512;
constexpr int kLpBnX = 96, kLpBnG = 128;
// epilogue: warp stores straight from registers (transposed outputs: one coalesced 128-byte
// column per instruction) or through one 4 KB shared-memory box per warp (row-major outputs,
// read back four 128-byte rows per instruction); no TMA stores, so no store-completion waits
// and 32 KB of boxes instead of 64 -- the difference deepens the operand rings (in-flight
// bytes per SM are what bound these latency-limited phases)
constexpr bool kLpLsuEpi = true;
constexpr int kLpRbStages = kLpLsuEpi ? 7 : 5, kLpGStages = kLpLsuEpi ? 4 : 3;
constexpr int kLpABytes = kBM * kBK * 4;                          // 16 KB raw A tile
constexpr int kLpXBBytes = kLpBnX * kBK * 4;                      // 12 KB resident k-block
constexpr int kLpResBytes = kRbMaxKt * 2 * kLpXBBytes;            // 72 KB
constexpr int kLpGBBytes = kLpBnG * kBK * 4;                      // 16 KB
constexpr int kLpGStage = kLpABytes + 2 * kLpGBBytes;             // 48 KB
constexpr int kLpRegion = std::max(kLpResBytes + kLpRbStages * kLpABytes, kLpGStages * kLpGStage);
constexpr int kLpEpiBytes = 8 * (kLpLsuEpi ? 1 : 2) * 4096;
constexpr int kLpSmem = kLpRegion + kLpEpiBytes + 1024 + 1024;
constexpr int kLpQ = 4;                                           // tile-queue slots
constexpr int kLpQCons = 32 + kConvA + 64 + 256;                  // queue readers: MMA, A conv, B conv, epilogue
constexpr int kLpAccStride = 128, kLpACol = 256;                  // TMEM: two accumulators, then 4 A stages
static_assert(kLpSmem <= 227 * 1024, "fused l_product shared memory");
static_assert(kLpACol + kTm3 * 64 <= 512, "fused l_product TMEM");

enum LpMapId { LP_XA, LP_XB, LP_KF, LP_KF_LO, LP_KI, LP_KI_LO, LP_HA_LD, LP_HB_LD, LP_HC_LD, LP_HA_ST, LP_HB_ST,
               LP_HC_ST, LP_C_ST, LP_NMAPS };
struct LpMaps {
  CUtensorMap m[LP_NMAPS];
};

struct LpShape {
  float* hA;          // slice-major stacks A-hat (P x I1 L), B-hat (P x L I2), C-hat (P x I1 x I2)
  float* hB;
  float* hC;
  float* C;           // the product, tube-major (I1 I2 x P)
  int P, I1, L, I2;
  int ktX, ktG;       // k-blocks of a transform / GEMM tile
  int num_m, num_n;   // 128-row blocks of A / C, 128-column blocks of B / C
  int nF, nG, nI;     // tiles per phase
  int total;
};

enum { LP_F = 0, LP_G = 1, LP_I = 2 };

struct LpTile {
  int kind;
  int op;     // F: 0 = A, 1 = B
  int m0;     // first row of the tile (tube for F / I, slice row for G)
  int n0;     // G: first column
  int b;      // G: slice q
  int sig;    // counter this tile completes (-1: none)
  int dep0, dep1;  // counters this tile waits for (-1: none)
};

// Tile list and dependency groups (counter indices; counter 0 is the claim counter):
//   F  [A rows block 0 | B columns block 0 | ... | B columns block num_n-1 | A rows block 1 | ...]
//      counters 1 + mb (A rows block mb, L tiles) and 1 + num_m + nb (B column block nb, L tiles)
//   G  (mb, nb) groups of P slices each, counter 1 + num_m + num_n + mb num_n + nb; needs A(mb), B(nb)
//   I  (mb, nb) groups of 128 tiles (rows of block mb, columns of block nb); needs G(mb, nb)
// so the first slice GEMMs need only A rows block 0 and B columns block 0 (the first 2 L of the
// F tiles), and the first inverse tiles only the slice GEMMs of (0, 0).
__device__ __forceinline__ LpTile lp_decode(const LpShape& s, int t) {
  LpTile d{0, 0, 0, 0, 0, -1, -1, -1};
  const int cA = 1, cB = 1 + s.num_m, cG = 1 + s.num_m + s.num_n;
  if (t < s.nF) {
    d.kind = LP_F;
    const int g = t / s.L, u = t - g * s.L;  // F group g: 0 = A(0), 1..num_n = B(nb), then A(1..)
    if (g >= 1 && g <= s.num_n) {
      const int nb = g - 1;
      d.op = 1;
      d.m0 = u * s.I2 + 128 * nb;  // B tubes (k = u, i2 in column block nb)
      d.sig = cB + nb;
    } else {
      const int mb = g == 0 ? 0 : g - s.num_n;
      d.m0 = 128 * (mb * s.L + u);  // A tubes of rows block mb are contiguous
      d.sig = cA + mb;
    }
  } else if (t < s.nF + s.nG) {
    d.kind = LP_G;
    const int u = t - s.nF, grp = u / s.P;
    const int mb = grp / s.num_n, nb = grp - mb * s.num_n;
    d.b = u - grp * s.P;
    d.m0 = 128 * mb;
    d.n0 = 128 * nb;
    d.sig = cG + grp;
    d.dep0 = cA + mb;
    d.dep1 = cB + nb;
  } else {
    d.kind = LP_I;
    const int u = t - s.nF - s.nG, grp = u >> 7;
    const int mb = grp / s.num_n, nb = grp - mb * s.num_n;
    d.m0 = (128 * mb + (u & 127)) * s.I2 + 128 * nb;  // C tubes (row i1, columns of block nb)
    d.dep0 = cG + grp;
  }
  return d;
}

__device__ __forceinline__ uint32_t ld_acquire(const int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// optional per-tile timeline (ltb_ctx_set_option LTB_OPT_TC_TIMELINE): dbg[0 .. 2 grid) CTA
// start / end; from kLpDbgBase, per CTA 32 tiles x 8 slots of %globaltimer:
//   0 tile id, 1 claimed, 2 dependencies met, 3 last TMA issued, 4 last MMA issued,
//   5 epilogue saw the accumulator, 6 epilogue done (all slots written by one lane each)
constexpr int kLpDbgBase = 512, kLpDbgTiles = 32;
// per k-block stamps of CTA 0 (first kLpDbgKb k-blocks, 4 slots): 0 TMA issued, 1 converter
// saw the tile land, 2 converter wrote TMEM, 3 MMA issued
constexpr int kLpDbgKbBase = kLpDbgBase + 148 * kLpDbgTiles * 8, kLpDbgKb = 48;
__device__ __forceinline__ void lp_kstamp(unsigned long long* dbg, int it, int slot) {
  if (!dbg || blockIdx.x != 0 || it >= kLpDbgKb) return;
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  dbg[kLpDbgKbBase + it * 4 + slot] = v;
}
__device__ __forceinline__ void lp_stamp(unsigned long long* dbg, int j, int slot, unsigned long long v = 0) {
  if (!dbg || j >= kLpDbgTiles) return;
  if (!v) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  dbg[kLpDbgBase + ((int64_t)blockIdx.x * kLpDbgTiles + j) * 8 + slot] = v;
}

// counters: [0] tile claims, then the dependency groups of lp_decode
__global__ void __launch_bounds__(kLpThreads, 1)
    lprod_fused_kernel(const __grid_constant__ LpMaps maps, LpShape sh, int* __restrict__ ctr,
                       unsigned long long* dbg) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* region =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* ebuf0 = region + kLpRegion;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(ebuf0 + kLpEpiBytes);  // [5] F / I ring: raw A landed
  uint64_t* rfree = rfull + kLpRbStages;                               // [5] raw A read by the converters
  uint64_t* gfull = rfree + kLpRbStages;                               // [4] G ring: A + B landed
  uint64_t* gfree = gfull + kLpGStages;                                // [4] MMAs of the G stage done
  uint64_t* tfull = gfree + kLpGStages;                                // [4] TMEM A stage (and B split) ready
  uint64_t* tfree = tfull + kTm3;                                      // [4] MMAs reading the TMEM stage done
  uint64_t* accf = tfree + kTm3;                                       // [2] accumulator ready
  uint64_t* acce = accf + 2;                                           // [2] accumulator drained
  uint64_t* bres = acce + 2;                                           // resident matrix landed
  uint64_t* qfull = bres + 1;                                          // [kLpQ] tile id published
  uint64_t* qfree = qfull + kLpQ;                                      // [kLpQ] tile id read by every role
  int* tq = reinterpret_cast<int*>(qfree + kLpQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kLpQ);
  auto res_hi = [&](int kt) { return region + kt * 2 * kLpXBBytes; };
  auto res_lo = [&](int kt) { return region + kt * 2 * kLpXBBytes + kLpXBBytes; };
  auto r_stage = [&](int s) { return region + kLpResBytes + s * kLpABytes; };
  auto g_stage = [&](int s) { return region + s * kLpGStage; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (dbg && threadIdx.x == 0) {
    unsigned long long tns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
    dbg[2 * blockIdx.x] = tns;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLpRbStages; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rfree[s], kConvA + 1);  // converters read it; the MMAs (F tiles: A hi from here) done
    }
    for (int s = 0; s < kLpGStages; ++s) {
      mbar_init(&gfull[s], 1);
      mbar_init(&gfree[s], 1);
    }
    for (int s = 0; s < kTm3; ++s) {
      mbar_init(&tfull[s], kConvA + 64);
      mbar_init(&tfree[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accf[a], 1);
      mbar_init(&acce[a], 256);
    }
    mbar_init(bres, 1);
    for (int s = 0; s < kLpQ; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qfree[s], kLpQCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < LP_NMAPS; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[i])) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // every role reads the same tile sequence from the queue
  int qi = 0;
  auto next_tile = [&]() -> int {
    const int slot = qi % kLpQ;
    mbar_wait(&qfull[slot], (qi / kLpQ) & 1);
    const int t = *reinterpret_cast<volatile int*>(&tq[slot]);
    mbar_arrive(&qfree[slot]);
    ++qi;
    return t;
  };
  // resident matrix of a transform tile: 0 = K (forward), 1 = Kinv
  auto res_of = [](int kind) { return kind == LP_I ? 1 : 0; };

  if (warp == 0) {
    // ---------------------------------------------------------------- claimer + TMA producer
    if (lane == 0) {
      int it_r = 0, it_g = 0, it_t = 0, cur = -1, res = -1;
      const int nAB = 1 + sh.num_m + sh.num_n;  // counters below nAB count F tiles (L per group)
      uint64_t ok = 0;                           // counters seen complete (at most 64)
      int jp = 0;
      for (;;) {
        int t = atomicAdd(ctr, 1);
        lp_stamp(dbg, jp, 1);
        if (t >= sh.total) t = -1;
        const int slot = qi % kLpQ;
        mbar_wait(&qfree[slot], ((qi / kLpQ) & 1) ^ 1);
        tq[slot] = t;
        mbar_arrive(&qfull[slot]);
        ++qi;
        if (t < 0) break;
        lp_stamp(dbg, jp, 0, (unsigned long long)t + 1);
        const LpTile d = lp_decode(sh, t);
        const bool gk = d.kind == LP_G;
        if ((cur == LP_G) != gk && cur >= 0) {
          // the region changes use: every MMA issued so far (readers of the ring, the
          // resident matrix and the B splits) must have completed
          for (int i = max(0, it_t - kTm3); i < it_t; ++i) mbar_wait(&tfree[i % kTm3], (i / kTm3) & 1);
          if (gk) res = -1;  // the G ring overwrites the resident matrix
        }
        cur = d.kind;
        if (!gk && res != res_of(d.kind)) {
          if (res >= 0)  // K -> Kinv without a G tile between: drain the resident's readers
            for (int i = max(0, it_t - kTm3); i < it_t; ++i) mbar_wait(&tfree[i % kTm3], (i / kTm3) & 1);
          res = res_of(d.kind);
          const CUtensorMap* kh = &maps.m[res ? LP_KI : LP_KF];
          const CUtensorMap* kl = &maps.m[res ? LP_KI_LO : LP_KF_LO];
          mbar_expect_tx(bres, sh.ktX * 2 * kLpXBBytes);
          for (int kt = 0; kt < sh.ktX; ++kt) {
            tma_load_3d(res_hi(kt), kh, bres, kt * kBK, 0, 0);
            tma_load_3d(res_lo(kt), kl, bres, kt * kBK, 0, 0);
          }
        }
        // dependencies (a group is complete once all 8 epilogue warps of each of its tiles signalled)
        bool waited = false;
        for (int k = 0; k < 2; ++k) {
          const int c = k ? d.dep1 : d.dep0;
          if (c < 0 || ((ok >> c) & 1)) continue;
          const int target = 8 * (c < nAB ? sh.L : sh.P);
          while ((int)ld_acquire(ctr + c) < target) __nanosleep(64);
          ok |= 1ull << c;
          waited = true;
        }
        if (waited) fence_proxy_async_global();
        lp_stamp(dbg, jp, 2);
        if (!gk) {
          const CUtensorMap* ma = &maps.m[d.kind == LP_I ? LP_HC_LD : (d.op ? LP_XB : LP_XA)];
          for (int kt = 0; kt < sh.ktX; ++kt, ++it_r, ++it_t) {
            const int s = it_r % kLpRbStages;
            mbar_wait(&rfree[s], ((it_r / kLpRbStages) & 1) ^ 1);
            mbar_expect_tx(&rfull[s], kLpABytes);
            if (d.kind == LP_F) {
              tma_load_3d(r_stage(s), ma, &rfull[s], kt * kBK, d.m0, 0);
            } else {  // C-hat is slice-major: an MN-major A, four unswizzled [32 k][32 rows] boxes
              for (int c = 0; c < kBM / 32; ++c) tma_load_3d(r_stage(s) + c * 4096, ma, &rfull[s], d.m0 + 32 * c, kt * kBK, 0);
            }
            lp_kstamp(dbg, it_t, 0);
          }
        } else {
          for (int kt = 0; kt < sh.ktG; ++kt, ++it_g, ++it_t) {
            const int s = it_g % kLpGStages;
            mbar_wait(&gfree[s], ((it_g / kLpGStages) & 1) ^ 1);
            mbar_expect_tx(&gfull[s], kLpABytes + kLpGBBytes);
            tma_load_3d(g_stage(s), &maps.m[LP_HA_LD], &gfull[s], kt * kBK, d.m0, d.b);
            for (int c = 0; c < kLpBnG / 32; ++c)
              tma_load_3d(g_stage(s) + kLpABytes + c * 4096, &maps.m[LP_HB_LD], &gfull[s], d.n0 + 32 * c, kt * kBK,
                          d.b);
            lp_kstamp(dbg, it_t, 0);
          }
        }
        lp_stamp(dbg, jp, 3);
        ++jp;
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idX = idesc_tf32(kLpBnX, false, false);
    constexpr uint32_t idG = idesc_tf32(kLpBnG, false, true);
    int it_g = 0, it_r = 0, it_t = 0, j = 0, nres = 0, res = -1;
    for (;;) {
      const int t = next_tile();
      if (t < 0) break;
      const LpTile d = lp_decode(sh, t);
      const bool gk = d.kind == LP_G;
      if (gk) res = -1;
      if (!gk && res != res_of(d.kind)) {  // the producer loaded a resident matrix for this tile
        res = res_of(d.kind);
        mbar_wait(bres, nres & 1);
        ++nres;
      }
      const int a = j & 1;
      mbar_wait(&acce[a], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(a * kLpAccStride);
      const int nk = gk ? sh.ktG : sh.ktX;
      for (int kt = 0; kt < nk; ++kt, ++it_t) {
        const int ts = it_t % kTm3;
        mbar_wait(&tfull[ts], (it_t / kTm3) & 1);
        tc_fence_after();
        if (lane == 0) lp_kstamp(dbg, it_t, 3);
        const uint32_t ahi = tmem + (uint32_t)(kLpACol + 64 * ts), alo = ahi + 32;
        // K-major A (F and G tiles): the raw fp32 tile in shared memory is the hi operand
        // (kind::tf32 reads the top 19 bits, i.e. trunc(x), as for B-hat below), so the
        // converters write only lo = round(x - trunc(x)) to TMEM
        if (gk) {
          const int s = it_g % kLpGStages;
          const uint64_t dah0 = umma_desc(smem_u32(g_stage(s)), 16u, 1024u, false);
          const uint64_t dbh0 = umma_desc(smem_u32(g_stage(s) + kLpABytes), g_mn_lbo, g_mn_sbo, true);
          const uint64_t dbl0 = umma_desc(smem_u32(g_stage(s) + kLpABytes + kLpGBBytes), g_mn_lbo, g_mn_sbo, true);
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint64_t kof = (uint64_t)((1024u * kk) >> 4), aof = (uint64_t)((32u * kk) >> 4);
            umma_tf32_w(dacc, dah0 + aof, dbh0 + kof, idG, (kt > 0 || kk > 0) ? 1u : 0u);
            umma_tf32_w(dacc, dah0 + aof, dbl0 + kof, idG, 1u);
            umma_tf32_ta_w(dacc, alo + 8 * kk, dbh0 + kof, idG, 1u);
          }
          umma_commit_w(&tfree[ts]);
          umma_commit_w(&gfree[s]);
          ++it_g;
        } else {
          const int s = it_r % kLpRbStages;
          const uint64_t dbh0 = umma_desc(smem_u32(res_hi(kt)), 16u, 1024u, false);
          const uint64_t dbl0 = umma_desc(smem_u32(res_lo(kt)), 16u, 1024u, false);
          if (d.kind == LP_F) {
            const uint64_t dah0 = umma_desc(smem_u32(r_stage(s)), 16u, 1024u, false);
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint64_t kof = (uint64_t)((32u * kk) >> 4);
              umma_tf32_w(dacc, dah0 + kof, dbh0 + kof, idX, (kt > 0 || kk > 0) ? 1u : 0u);
              umma_tf32_w(dacc, dah0 + kof, dbl0 + kof, idX, 1u);
              umma_tf32_ta_w(dacc, alo + 8 * kk, dbh0 + kof, idX, 1u);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint64_t kof = (uint64_t)((32u * kk) >> 4);
              umma_tf32_ta_w(dacc, ahi + 8 * kk, dbh0 + kof, idX, (kt > 0 || kk > 0) ? 1u : 0u);
              umma_tf32_ta_w(dacc, ahi + 8 * kk, dbl0 + kof, idX, 1u);
              umma_tf32_ta_w(dacc, alo + 8 * kk, dbh0 + kof, idX, 1u);
            }
          }
          umma_commit_w(&tfree[ts]);
          umma_commit_w(&rfree[s]);  // the raw stage may be refilled once these MMAs completed
          ++it_r;
        }
        if (kt == nk - 1) {
          umma_commit_w(&accf[a]);
          if (lane == 0) lp_stamp(dbg, j, 4);
        }
        __syncwarp();
      }
      ++j;
    }
  } else if (warp < 6) {
    // ---------------------------------------------------------------- A -> TMEM (hi, lo)
    const int q = warp & 3, row = 32 * q + lane;
    int it_r = 0, it_g = 0, it_t = 0;
    for (;;) {
      const int t = next_tile();
      if (t < 0) break;
      const LpTile d = lp_decode(sh, t);
      const bool gk = d.kind == LP_G;
      const int nk = gk ? sh.ktG : sh.ktX;
      for (int kt = 0; kt < nk; ++kt, ++it_t) {
        uint32_t hi[32], lo[32];
        const unsigned char* ab;
        int s;
        if (gk) {
          s = it_g % kLpGStages;
          mbar_wait(&gfull[s], (it_g / kLpGStages) & 1);
          ab = g_stage(s);
          ++it_g;
        } else {
          s = it_r % kLpRbStages;
          mbar_wait(&rfull[s], (it_r / kLpRbStages) & 1);
          ab = r_stage(s);
          ++it_r;
        }
        if (threadIdx.x == 64) lp_kstamp(dbg, it_t, 1);
        const bool kmaj = d.kind != LP_I;
        if (kmaj) {  // 128B-swizzled K-major rows: 16-byte chunk c of row r at c ^ (r & 7); lo only
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(ab + row * 128 + ((c ^ (row & 7)) << 4));
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) lo[4 * c + e] = __float_as_uint(tf32_round(x[e] - tf32_trunc(x[e])));
          }
        } else {  // unswizzled [k][32 rows] boxes
          const float* cb = reinterpret_cast<const float*>(ab + (row >> 5) * 4096) + (row & 31);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = cb[32 * k];
            const float h = tf32_trunc(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(tf32_round(x - h));
          }
        }
        if (!gk) mbar_arrive(&rfree[s]);  // the raw tile is in registers: the TMA may refill it
        const int ts = it_t % kTm3;
        mbar_wait(&tfree[ts], ((it_t / kTm3) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tq4 = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(kLpACol + 64 * ts);
        if (!kmaj) tmem_st32(tq4, hi);
        tmem_st32(tq4 + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        if (threadIdx.x == 64) lp_kstamp(dbg, it_t, 2);
        mbar_arrive(&tfull[ts]);
      }
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- B-hat lo split (G tiles)
    const int cv = threadIdx.x - 192;  // 0 .. 63
    int it_g = 0, it_t = 0;
    for (;;) {
      const int t = next_tile();
      if (t < 0) break;
      const LpTile d = lp_decode(sh, t);
      const bool gk = d.kind == LP_G;
      const int nk = gk ? sh.ktG : sh.ktX;
      for (int kt = 0; kt < nk; ++kt, ++it_t) {
        if (gk) {
          const int s = it_g % kLpGStages;
          mbar_wait(&gfull[s], (it_g / kLpGStages) & 1);
          const float4* bh = reinterpret_cast<const float4*>(g_stage(s) + kLpABytes);
          float4* bl = reinterpret_cast<float4*>(g_stage(s) + kLpABytes + kLpGBBytes);
#pragma unroll 4
          for (int i = cv; i < kLpGBBytes / 16; i += 64) {
            const float4 x = bh[i];
            const float4 h = make_float4(tf32_trunc(x.x), tf32_trunc(x.y), tf32_trunc(x.z), tf32_trunc(x.w));
            bl[i] = make_float4(tf32_round(x.x - h.x), tf32_round(x.y - h.y), tf32_round(x.z - h.z),
                                tf32_round(x.w - h.w));
          }
          fence_proxy_async();
          ++it_g;
        }
        // the TMEM stage's previous MMAs are done before this k-block's arrival counts
        const int ts = it_t % kTm3;
        mbar_wait(&tfree[ts], ((it_t / kTm3) & 1) ^ 1);
        mbar_arrive(&tfull[ts]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (TMA tensor stores)
    const int q = warp & 3, half = (warp - 8) >> 2;
    unsigned char* ebuf = ebuf0 + (warp - 8) * (kLpLsuEpi ? 1 : 2) * 4096;
    int nbox = 0, j = 0;
    // completion signals are deferred: a warp adds its finished tiles of one group to the
    // group's counter only when its next tile belongs to another group (or it exits) -- one
    // fence per group, not per tile.  The flush happens before the next tile's accumulator
    // wait, so a producer blocked on the group never waits on this warp.
    int* pend_ctr = nullptr;
    int pend_n = 0;
    auto flush = [&]() {
      if (pend_n) {
        __syncwarp();
        if (lane == 0) {
          if constexpr (kLpLsuEpi) {
            // no separate fence: red.release orders the warp's stores (made visible to this
            // lane by the __syncwarp above; release is cumulative), and the consumer's
            // ld.acquire + fence.proxy.async orders them before its TMA loads
          } else {
            bulk_wait_all();
            fence_proxy_async_global();
          }
          red_release_add(pend_ctr, pend_n);
        }
        __syncwarp();
        pend_n = 0;
      }
    };
    for (;;) {
      const int t = next_tile();
      if (t < 0) break;
      const LpTile d = lp_decode(sh, t);
      int* my_ctr = d.sig >= 0 ? ctr + d.sig : nullptr;
      if (my_ctr != pend_ctr) flush();
      const int a = j & 1;
      mbar_wait(&accf[a], (j >> 1) & 1);
      if (warp == 8 && lane == 0) lp_stamp(dbg, j, 5);
      tc_fence_after();
      const int ct = d.kind == LP_F;
      const int bn = d.kind == LP_G ? kLpBnG : kLpBnX;
      const int ncol = d.kind == LP_G ? sh.I2 : sh.P;
      const int rows = d.kind == LP_G ? sh.I1 : (d.kind == LP_I ? sh.I1 * sh.I2 : (d.op ? sh.L * sh.I2 : sh.I1 * sh.L));
      const CUtensorMap* mc =
          &maps.m[d.kind == LP_G ? LP_HC_ST : (d.kind == LP_I ? LP_C_ST : (d.op ? LP_HB_ST : LP_HA_ST))];
      const int row0 = d.m0 + 32 * q;
#pragma unroll 1
      for (int c0 = 32 * half; c0 < bn && d.n0 + c0 < ncol; c0 += 64) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * kLpAccStride + c0), r);
        if constexpr (kLpLsuEpi) {
          if (ct) {
            // transposed output (slice-major A-hat / B-hat): column n of the chunk is 32
            // consecutive tubes = one coalesced 128-byte store per instruction
            float* out = d.op ? sh.hB : sh.hA;
            const int64_t ld = rows;
            if (row0 + lane < rows) {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (c0 + jj < ncol) out[(int64_t)(c0 + jj) * ld + row0 + lane] = __uint_as_float(r[jj]);
            }
          } else {
            // row-major output: rows through the box, read back as four 128-byte rows per instruction
            unsigned char* box = ebuf;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              *reinterpret_cast<float4*>(box + lane * 128 + ((jj ^ (lane & 7)) << 4)) =
                  make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                              __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
            __syncwarp();
            float* out = d.kind == LP_G ? sh.hC + (int64_t)d.b * sh.I1 * sh.I2 : sh.C;
            const int64_t ld = ncol;
            const int gc = d.n0 + c0 + 4 * (lane & 7);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rr = 4 * i + (lane >> 3), gr = row0 + rr;
              const float4 v = *reinterpret_cast<const float4*>(box + rr * 128 + (((lane & 7) ^ (rr & 7)) << 4));
              if (gr < rows) {
                float* dst = out + (int64_t)gr * ld + gc;
                if (gc + 3 < ncol) {
                  *reinterpret_cast<float4*>(dst) = v;
                } else {
                  const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (gc + u < ncol) dst[u] = e[u];
                }
              }
            }
            __syncwarp();
          }
          ++nbox;
          continue;
        }
        unsigned char* box = ebuf + (nbox & 1) * 4096;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
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
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && row0 < rows) {
          if (!ct)
            tma_store_3d(mc, box, d.n0 + c0, row0, d.b);
          else
            tma_store_3d(mc, box, row0, d.n0 + c0, 0);
          bulk_commit();
        }
        ++nbox;
      }
      tc_fence_before();
      mbar_arrive(&acce[a]);  // the accumulator is in registers / boxes: the MMA may reuse it
      if (my_ctr) {
        pend_ctr = my_ctr;
        ++pend_n;
      }
      if (warp == 8 && lane == 0) lp_stamp(dbg, j, 6);
      ++j;
    }
    flush();
    if (!kLpLsuEpi && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  // the last CTA to finish zeroes the counters for the next launch: by then every CTA has made
  // its final claim and no producer polls a group counter any more
  if (threadIdx.x == 0) {
    const int nctr = 1 + sh.num_m + sh.num_n + sh.num_m * sh.num_n;
    __threadfence();
    if (atomicAdd(ctr + nctr, 1) == (int)gridDim.x - 1) {
      for (int i = 0; i <= nctr; ++i) ctr[i] = 0;
      __threadfence();
    }
  }
  if (dbg && threadIdx.x == 0) {
    unsigned long long tns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
    dbg[2 * blockIdx.x + 1] = tns;
  }
}

}  // namespace

// fp32 real-spec *_L product on device buffers in one launch (see the header comment).
// A: I1 x L x trailing, B: L x I2 x trailing, C: I1 x I2 x trailing (tube-major, C-order);
// ws: lprod_fused_ws_bytes() bytes (the three slice-major stacks and the counters).
// LTB_EUNSUPPORTED when the shape or the spec does not fit (the caller runs three launches).
int64_t ltb_lprod_fused_ws_bytes(int64_t P, int64_t I1, int64_t L, int64_t I2) {
  return 4 * P * (I1 * L + L * I2 + I1 * I2) + 4 * 64 + 256;
}

int ltb_lprod_fused_f32(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, const float* A,
                        const float* B, float* C, void* ws, bool ws_clean) {
  const int64_t P = spec->P;
  if (spec->is_complex || !spec->d_kron[0] || !spec->d_kron[1] || spec->nmodes == 0) return LTB_EUNSUPPORTED;
  if (P < 8 || P > kLpBnX || P % 4 || I1 % 128 || I2 % 128 || I1 < 128 || I2 < 128 || L % 4 || L < 8 ||
      1 + I1 / 128 + I2 / 128 + (I1 / 128) * (I2 / 128) > 64)
    return LTB_EUNSUPPORTED;
  if (I1 * L >= (1ll << 31) || L * I2 >= (1ll << 31) || I1 * I2 >= (1ll << 31)) return LTB_EUNSUPPORTED;
  LpShape sh{};
  sh.P = (int)P;
  sh.I1 = (int)I1;
  sh.L = (int)L;
  sh.I2 = (int)I2;
  sh.ktX = (int)((P + kBK - 1) / kBK);
  sh.ktG = (int)((L + kBK - 1) / kBK);
  sh.num_m = (int)(I1 / 128);
  sh.num_n = (int)(I2 / 128);
  sh.nF = (sh.num_m + sh.num_n) * sh.L;
  sh.nG = sh.num_m * sh.num_n * sh.P;
  sh.nI = sh.num_m * sh.num_n * 128;
  sh.total = sh.nF + sh.nG + sh.nI;
  float* hA = (float*)ws;
  float* hB = hA + P * I1 * L;
  float* hC = hB + P * L * I2;
  int* ctr = (int*)(hC + P * I1 * I2);
  sh.hA = hA;
  sh.hB = hB;
  sh.hC = hC;
  sh.C = C;
  const float* K = spec->d_kron[0];
  const float* Ki = spec->d_kron[1];
  LpMaps maps;
  CUtensorMap* m = maps.m;
  const int64_t NA = I1 * L, NB = L * I2, NC = I1 * I2;
  bool ok = make_map(&m[LP_XA], A, P, NA, 1, P, 0, kBM) && make_map(&m[LP_XB], B, P, NB, 1, P, 0, kBM) &&
            make_map(&m[LP_KF], K, P, P, 1, P, 0, kLpBnX) && make_map(&m[LP_KF_LO], K + P * P, P, P, 1, P, 0, kLpBnX) &&
            make_map(&m[LP_KI], Ki, P, P, 1, P, 0, kLpBnX) &&
            make_map(&m[LP_KI_LO], Ki + P * P, P, P, 1, P, 0, kLpBnX) &&
            make_map(&m[LP_HA_LD], hA, L, I1, P, L, NA, kBM) && make_map(&m[LP_HB_LD], hB, I2, L, P, I2, NB, kBK, 1) &&
            make_map(&m[LP_HC_LD], hC, NC, P, 1, NC, 0, kBK, 2) && make_map(&m[LP_HA_ST], hA, NA, P, 1, NA, 0, 32) &&
            make_map(&m[LP_HB_ST], hB, NB, P, 1, NB, 0, 32) && make_map(&m[LP_HC_ST], hC, I2, I1, P, I2, NC, 32) &&
            make_map(&m[LP_C_ST], C, P, NC, 1, P, 0, 32);
  if (!ok) return LTB_EUNSUPPORTED;
  LTB_TRY(ensure_smem(ctx, lprod_fused_kernel, kLpSmem));
  // counters (and the exit counter): zero unless the caller guarantees the workspace is fresh
  // from a zero fill or from a completed launch (the kernel zeroes them on exit)
  if (!ws_clean)
    LTB_CUDA_TRY(ctx, cudaMemsetAsync(ctr, 0, sizeof(int) * (2 + sh.num_m + sh.num_n + sh.num_m * sh.num_n),
                                      ctx->stream));
  const int grid = (int)std::min<int64_t>(sh.total, ctx->num_sms);
  lprod_fused_kernel<<<grid, kLpThreads, kLpSmem, ctx->stream>>>(maps, sh, ctr, ctx->opt_tc_timeline);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}
