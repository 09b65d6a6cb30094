// tcgen05 (5th-gen tensor core) GEMM in 3xFP16 for sm_100a.
//
//   C = epi(alpha * A . B^T)      A: (M, K) fp32, B: (N, K), both K-major
//
// fp32-faithful on the fp16 tensor pipe (twice the tf32 rate): each operand
// x is split into hi = fp16(x) and lo = fp16(x - hi) (11 + 11 significant
// bits), and the product is accumulated as hi.hi + hi.lo + lo.hi in fp32 in
// TMEM (the dropped lo.lo term is ~2^-22 relative).  B operands that are
// weights or the encoder's K / V^T arrive pre-split and pre-scaled by a
// power of two s (s.w = hi + lo keeps lo in fp16's normal range; the
// epilogue's alpha carries 1/s).  Activations (A, and B on the trunk's
// reassociated products) are split on chip, unscaled: fp16's subnormal
// floor (2^-25 absolute) is far below the beam-score tolerance for O(1)
// activations.  Range: |activation| < 65504, |s.B| < 65504 (conversions
// saturate).  This keeps the beam scores within ~1e-6 of float64, which the
// list-identity parity rule needs (SURVEY §7 hard part 1); plain TF32 / BF16
// / FP16 inputs reorder most beam lists.
//
// Pipeline per CTA (persistent; one 128 x BN output tile at a time, K in
// 32-element stages):
//   warp 0     TMA producer: fp32 A tile (SWIZZLE_128B) and the B tile --
//              fp16 hi + lo (SWIZZLE_64B) or fp32 (SWIZZLE_128B) -> smem
//   warps 2-5  converters: fp32 -> fp16 hi / lo tiles in the UMMA K-major
//              SWIZZLE_64B layout, fence.proxy.async, arrive
//   warp 1     TMEM allocator + single-thread MMA issuer: 3 tcgen05.mma
//              (kind::f16, 128 x BN x 16) per 16-deep k-step; tcgen05.commit
//              frees the stage
//   warps 6-9  epilogue: tcgen05.ld 32x32b the double-buffered 128 x BN fp32
//              accumulator, bias / GELU / residual / gate / K|V^T split, store
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include <algorithm>

#include "gemm.cuh"
#include "gemm_tc.cuh"

namespace gr {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;           // k per stage: one 128-B fp32 row, two 16-deep MMA k-steps
constexpr int kConvWarps = 4;    // warps 2 .. 2 + kConvWarps - 1
constexpr int kEpiWarp0 = 2 + kConvWarps;
// two epilogue warps per TMEM lane quarter: with BN = 256 they drain the
// accumulator's column halves in parallel (one warp per SMSP was latency-bound
// on the heavier epilogues)
#ifndef GR_TC_EPI_WARPS
#define GR_TC_EPI_WARPS 8
#endif
constexpr int kEpiWarps = GR_TC_EPI_WARPS;
constexpr int kTcThreads = 32 * (kEpiWarp0 + kEpiWarps);

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}

// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cluster_addr(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// arrive on an mbarrier of another CTA of the cluster (shared::cluster address)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}

// CTA-pair load: lands in this CTA's shared memory, completes on the pair
// leader's mbarrier (shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t cbar,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cbar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// commit to the mbarrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major SWIZZLE_64B smem matrix descriptor (rows of 64 B = 32 fp16, 8-row
// core-matrix atoms of 512 B, consecutive atoms sbo bytes apart):
// start>>4 | LBO=1 (16 B) | SBO | version 1 | layout 4
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace

// x (scaled by s) -> fp16 hi + lo with s.x == hi + lo to ~2^-22 (saturating)
__device__ __forceinline__ void split_f16x2(float x0, float x1, float s, uint32_t &hi,
                                            uint32_t &lo) {
  const float2 v = make_float2(x0 * s, x1 * s);
  const __half2 h = __float22half2_rn(v);
  const float2 hf = __half22float2(h);
  const __half2 l = __float22half2_rn(make_float2(v.x - hf.x, v.y - hf.y));
  hi = *reinterpret_cast<const uint32_t *>(&h);
  lo = *reinterpret_cast<const uint32_t *>(&l);
}

__device__ __forceinline__ void dbg_stamp(long long *dbg, int slot) {
  if (!dbg) return;
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  dbg[blockIdx.x * 8 + slot] = t;
}

struct TileInfo {
  int m0, n0, M, N, K;
  int a_row, a_k, b_row, b_k;  // operand bases (rows, k) of the tile's group
  int c_row;                   // C row of tile row 0 (of tile column 0 when transposed)
  bool valid;
};

// tile -> (group, m-tile, n-tile); identical in every warp role
// (bm: tile rows -- 2 BM for a CTA pair, whose CTA `moff / BM` owns rows
// [m0 + moff, m0 + moff + BM) of the pair's tile)
__device__ __forceinline__ TileInfo tile_info(const TcArgs &a, int tile, int tiles_m, int tiles_n,
                                              int bn, int bm = BM, int moff = 0) {
  TileInfo ti;
  const int per_g = tiles_m * tiles_n;
  const int g = tile / per_g, r = tile - g * per_g;
  const int tm = r / tiles_n, tn = r - tm * tiles_n;
  ti.M = a.M; ti.N = a.N; ti.K = a.K;
  ti.a_row = 0; ti.a_k = 0; ti.b_row = 0; ti.b_k = 0; ti.c_row = 0;
  if (a.g_rows) {
    if (a.mode == GM_QK_T) {  // M = the request's keys, N = its rows
      ti.M = a.g_ctx_len[g];
      ti.a_row = a.g_ctx_off[g];
      ti.N = a.g_rows[g];
      ti.b_row = a.g_row_off[g];
      ti.c_row = a.g_row_off[g];
    } else if (a.mode == GM_PV_T) {  // M = dims, N = rows, K = the request's keys
      ti.a_k = a.g_ctx_off[g];
      ti.N = a.g_rows[g];
      ti.b_row = a.g_row_off[g];
      ti.K = a.g_ctx_len[g];
      ti.c_row = a.g_row_off[g];
    } else {
      ti.a_row = a.g_row_off[g];
      ti.c_row = a.g_row_off[g];
      ti.M = a.g_rows[g];
      if (a.mode == GM_QK) {
        ti.N = a.g_ctx_len[g];
        ti.b_row = a.g_ctx_off[g];
      } else if (a.mode == GM_PV) {
        ti.K = a.g_ctx_len[g];
        ti.b_k = a.g_ctx_off[g];
      }
    }
  }
  ti.m0 = tm * bm + moff;
  ti.n0 = tn * bn;
  ti.valid = tm * bm < ti.M && ti.n0 < ti.N;
  return ti;
}

// In-place split of a landed fp32 tile [rows][32] (SWIZZLE_128B, as TMA
// writes it) into the fp16 hi / lo UMMA operand tiles (SWIZZLE_64B): the
// 1024 B of every 8-row group become its 512-B hi atom followed by its 512-B
// lo atom, so each group converts locally (one warp, no block barrier) and
// the operand descriptors step 1024 B between atoms.  A lane handles 8
// consecutive k of one row (two 16-B fp32 chunks -> one 16-B hi + one lo).
__device__ __forceinline__ void convert_groups(unsigned char *tile, int rows, int warp_idx,
                                               int n_warps) {
  const int lane = threadIdx.x & 31, rr = lane >> 2, c8 = lane & 3;
  for (int grp = warp_idx; grp < rows / 8; grp += n_warps) {
    unsigned char *g = tile + grp * 1024;
    const float4 x0 = *reinterpret_cast<const float4 *>(g + rr * 128 + (((2 * c8) ^ rr) << 4));
    const float4 x1 = *reinterpret_cast<const float4 *>(g + rr * 128 + (((2 * c8 + 1) ^ rr) << 4));
    uint4 h, l;
    split_f16x2(x0.x, x0.y, 1.f, h.x, l.x);
    split_f16x2(x0.z, x0.w, 1.f, h.y, l.y);
    split_f16x2(x1.x, x1.y, 1.f, h.z, l.z);
    split_f16x2(x1.z, x1.w, 1.f, h.w, l.w);
    __syncwarp();  // the group's fp32 is in registers before it is overwritten
    const int o = rr * 64 + ((c8 ^ (rr >> 1)) << 4);
    *reinterpret_cast<uint4 *>(g + o) = h;
    *reinterpret_cast<uint4 *>(g + 512 + o) = l;
  }
}

// Persistent, warp-specialised: each CTA walks tiles blockIdx.x, +gridDim.x, ...
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile j overlap
// the MMAs of tile j+1.  BSPLIT: B arrives as pre-split fp16 hi / lo.
// PAIR (both operands pre-split): a cluster of two CTAs on one TPC computes
// 256 x BN tiles with tcgen05.mma.cta_group::2 issued by the leader; each CTA
// loads its 128 rows of A and half of the B tile (BN / 2 rows), so per SM the
// shared-memory operand traffic per flop drops by a third.  Stage-full
// barriers live in the leader (both CTAs' TMA bytes complete there), stage-
// free and accumulator-ready barriers are multicast commits to both CTAs,
// and both CTAs' epilogues release the accumulator on the leader's barrier.
template <int BN, int STAGES, int EPI, bool BSPLIT, bool ASPLIT, bool PAIR = false>
__global__ void __launch_bounds__(kTcThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmAlo,
               TcArgs a, int tiles_m, int tiles_n, int n_tiles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int A32 = BM * BK * 4;   // fp32 landing tile split in place (hi / lo atoms),
                                     // or (ASPLIT) the fp16 hi tile then the lo tile
  constexpr int A16 = BM * BK * 2;
  static_assert(!PAIR || (BSPLIT && ASPLIT), "CTA pairs take pre-split operands");
  constexpr int BNL = PAIR ? BN / 2 : BN;  // B rows loaded by this CTA
  constexpr int B16 = BNL * BK * 2;  // pre-split B: fp16 hi tile, then lo tile
  constexpr int B32 = BN * BK * 4;   // fp32 B landing tile, split in place
  // stage: [A][B]; A (and an fp32 B) hold interleaved 512-B hi / lo atoms
  constexpr int STAGE_BYTES = A32 + (BSPLIT ? 2 * B16 : B32);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *conv = full + STAGES;
  uint64_t *empty = conv + STAGES;
  uint64_t *accf = empty + STAGES;  // [2] accumulator ready
  uint64_t *acce = accf + 2;        // [2] accumulator drained
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) dbg_stamp(a.dbg, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kConvWarps);
      mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&accf[j], 1);
      mbar_init(&acce[j], PAIR ? 2 * kEpiWarps : kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the leader's barriers exist before any peer traffic
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) dbg_stamp(a.dbg, 1);
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int tstep = PAIR ? gridDim.x / 2 : gridDim.x;  // tiles are per pair
  const int tfirst = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int moff = (int)rank * BM;
  constexpr int TBM = PAIR ? 2 * BM : BM;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int kg = 0;
      for (int tile = tfirst; tile < n_tiles; tile += tstep) {
        const TileInfo ti = tile_info(a, tile, tiles_m, tiles_n, BN, TBM, moff);
        if (!ti.valid) continue;
        const int nk = (ti.K + BK - 1) / BK;
        for (int kt = 0; kt < nk; ++kt, ++kg) {
          const int s = kg % STAGES;
          if (kg >= STAGES) mbar_wait(&empty[s], ((kg / STAGES) - 1) & 1);
          unsigned char *st = smem + s * STAGE_BYTES;
          if constexpr (PAIR) {
            if (kg == 0) dbg_stamp(a.dbg, 2);
            const uint32_t fb = cluster_addr(&full[s], 0);
            if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);  // both CTAs' bytes
            const int ak = ti.a_k + kt * BK, bk = ti.b_k + kt * BK;
            tma_load_2d_pair(st, &tmA, fb, ak, ti.a_row + ti.m0);
            tma_load_2d_pair(st + A16, &tmAlo, fb, ak, ti.a_row + ti.m0);
            tma_load_2d_pair(st + A32, &tmB, fb, bk, ti.b_row + ti.n0 + (int)rank * BNL);
            tma_load_2d_pair(st + A32 + B16, &tmBlo, fb, bk, ti.b_row + ti.n0 + (int)rank * BNL);
            continue;
          }
          if (kg == 0) dbg_stamp(a.dbg, 2);
          mbar_expect_tx(&full[s], A32 + (BSPLIT ? 2 * B16 : B32));
          tma_load_2d(st, &tmA, &full[s], ti.a_k + kt * BK, ti.a_row + ti.m0);
          if (ASPLIT) tma_load_2d(st + A16, &tmAlo, &full[s], ti.a_k + kt * BK, ti.a_row + ti.m0);
          if (BSPLIT) {
            unsigned char *bh = st + A32;
            tma_load_2d(bh, &tmB, &full[s], ti.b_k + kt * BK, ti.b_row + ti.n0);
            tma_load_2d(bh + B16, &tmBlo, &full[s], ti.b_k + kt * BK, ti.b_row + ti.n0);
          } else {
            tma_load_2d(st + A32, &tmB, &full[s], ti.b_k + kt * BK, ti.b_row + ti.n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---- MMA issuer (the pair's leader)
      // kind::f16: D f32 (bit 4), A / B fp16 (format 0), both K-major, N >> 3, M >> 4
      constexpr uint32_t idesc =
          (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);
      int kg = 0, j = 0;
      for (int tile = tfirst; tile < n_tiles; tile += tstep) {
        const TileInfo ti = tile_info(a, tile, tiles_m, tiles_n, BN, TBM, moff);
        if (!ti.valid) continue;
        const int acc = j & 1;
        if (j >= 2) mbar_wait(&acce[acc], ((j >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem + (uint32_t)(acc * BN);
        const int nk = (ti.K + BK - 1) / BK;
        for (int kt = 0; kt < nk; ++kt, ++kg) {
          const int s = kg % STAGES;
          mbar_wait(PAIR ? &full[s] : &conv[s], (kg / STAGES) & 1);
          if (kg == 0) dbg_stamp(a.dbg, 3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
          // in-place split: interleaved hi / lo atoms 1024 B apart; ASPLIT: two tiles
          const uint32_t a_hi = st, a_lo = ASPLIT ? st + A16 : st + 512;
          constexpr uint32_t a_sbo = ASPLIT ? 512 : 1024;
          const uint32_t b_hi = st + A32, b_lo = BSPLIT ? b_hi + B16 : b_hi + 512;
          constexpr uint32_t b_sbo = BSPLIT ? 512 : 1024;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t off = k * 32;  // 16 fp16 = 32 B along the swizzled row
            const uint32_t acc0 = (kt > 0 || k > 0) ? 1u : 0u;
            if constexpr (PAIR) {
              mma_f16_pair(d_tmem, sw64_desc(a_lo + off, a_sbo), sw64_desc(b_hi + off, b_sbo), idesc, acc0);
              mma_f16_pair(d_tmem, sw64_desc(a_hi + off, a_sbo), sw64_desc(b_lo + off, b_sbo), idesc, 1u);
              mma_f16_pair(d_tmem, sw64_desc(a_hi + off, a_sbo), sw64_desc(b_hi + off, b_sbo), idesc, 1u);
            } else {
              mma_f16(d_tmem, sw64_desc(a_lo + off, a_sbo), sw64_desc(b_hi + off, b_sbo), idesc, acc0);
              mma_f16(d_tmem, sw64_desc(a_hi + off, a_sbo), sw64_desc(b_lo + off, b_sbo), idesc, 1u);
              mma_f16(d_tmem, sw64_desc(a_hi + off, a_sbo), sw64_desc(b_hi + off, b_sbo), idesc, 1u);
            }
          }
          if (PAIR)
            mma_commit_pair(&empty[s]);  // frees the stage in both CTAs
          else
            mma_commit(&empty[s]);  // frees the stage when these MMAs complete
        }
        if (PAIR)
          mma_commit_pair(&accf[acc]);
        else
          mma_commit(&accf[acc]);
        ++j;
      }
      dbg_stamp(a.dbg, 4);
    }
  } else if (warp < kEpiWarp0) {
    // ---- converters: landed fp32 tiles -> fp16 hi / lo operand tiles
    const int cw = warp - 2;  // converter warp index
    int kg = 0;
    for (int tile = blockIdx.x; !PAIR && tile < n_tiles; tile += gridDim.x) {
      const TileInfo ti = tile_info(a, tile, tiles_m, tiles_n, BN);
      if (!ti.valid) continue;
      const int nk = (ti.K + BK - 1) / BK;
      for (int kt = 0; kt < nk; ++kt, ++kg) {
        const int s = kg % STAGES;
        mbar_wait(&full[s], (kg / STAGES) & 1);
        unsigned char *st = smem + s * STAGE_BYTES;
        if (!ASPLIT) convert_groups(st, BM, cw, kConvWarps);
        if (!BSPLIT) convert_groups(st + A32, BN, cw, kConvWarps);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ---- epilogue: TMEM -> registers -> smem (transpose) -> coalesced global
    // A lane owns a row after tcgen05.ld; each 32-column chunk is staged
    // through a padded per-warp buffer so that global traffic (C, R, bias,
    // gate, K) runs with lanes along columns: one 128-B line per access.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    float *ebuf = reinterpret_cast<float *>(smem + STAGES * STAGE_BYTES + 256) +
                  (warp - kEpiWarp0) * 32 * 33;
    int j = 0;
    for (int tile = tfirst; tile < n_tiles; tile += tstep) {
      const TileInfo ti = tile_info(a, tile, tiles_m, tiles_n, BN, TBM, moff);
      if (!ti.valid) continue;
      const int acc = j & 1;
      mbar_wait(&accf[acc], (j >> 1) & 1);
      if (j == 0 && warp == kEpiWarp0 && lane == 0) dbg_stamp(a.dbg, 5);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int rbase = ti.m0 + q * 32;  // this warp's 32 rows (tile M side)
      const int nrows = min(32, ti.M - rbase);
      const int N = ti.N;
      // EPI_STORE_LSE: this lane's row, current 128 columns: max, sum, top-2
      float pm = -INFINITY, ps = 0.f, pt1 = -INFINITY, pt2 = -INFINITY;
      // this warp's chunks: with two warps per lane quarter and BN = 256 each
      // drains one 128-column half (whole log-sum-exp parts); narrower tiles
      // leave the second warp idle
      constexpr int NC = BN / 32;
      // (LSE parts need a warp's four consecutive chunks: 128 columns)
      constexpr bool halves =
          kEpiWarps == 8 && (NC >= 8 || (NC >= 2 && EPI != EPI_STORE_LSE));
      const int eh = (warp - kEpiWarp0) >> 2;
      const int c_begin = halves ? eh * (NC / 2) : 0;
      const int c_end = halves ? c_begin + NC / 2 : (eh == 0 ? NC : 0);
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
        const int col0 = ti.n0 + c * 32;
        if (nrows <= 0 || col0 >= N) continue;  // warp-uniform
        if (EPI == EPI_STORE_LSE) {  // online (max, sum exp) over the row-per-lane registers
          // four independent accumulators (no 32-long dependency chains);
          // exp as ex2.approx of a pre-scaled argument (rel. error ~2^-22)
          constexpr float kL2e = 1.4426950408889634f;
          float x[32];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) x[jj] = col0 + jj < N ? v[jj] * a.alpha : -INFINITY;
          float m4[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
          for (int jj = 4; jj < 32; ++jj) m4[jj & 3] = fmaxf(m4[jj & 3], x[jj]);
          const float cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          const float nm = fmaxf(pm, cm);  // finite: col0 < N
          const float nl = nm * kL2e;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) s4[jj & 3] += exp2f(fmaf(x[jj], kL2e, -nl));
          const float cs = (s4[0] + s4[1]) + (s4[2] + s4[3]);
          ps = (pm == -INFINITY ? 0.f : ps * exp2f((pm - nm) * kL2e)) + cs;
          pm = nm;
          // window proxies: the maxima of the part's two 64-column halves
          // (each a real candidate value, as the selection requires)
          if ((c & 3) < 2)
            pt1 = fmaxf(pt1, cm);
          else
            pt2 = fmaxf(pt2, cm);
          if ((c & 3) == 3 || col0 + 32 >= N) {
            if (lane < nrows)
              a.lse_part[((long long)ti.c_row + rbase + lane) * a.lse_ld + col0 / 128] =
                  make_float4(pm, ps, pt1, pt2);
            pm = -INFINITY;
            ps = 0.f;
            pt1 = pt2 = -INFINITY;
          }
        }
        if (EPI == EPI_STORE_T || EPI == EPI_STORE_T_SPLIT) {
          // C[c_row + n][m]: lanes (m) are contiguous in every stored row
          const int m = rbase + lane;
          if (lane < nrows) {
            const long long o0 = (long long)ti.c_row * a.ldc + m;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (col0 + jj < N) {
                const float x = v[jj] * a.alpha;
                const long long o = o0 + (long long)(col0 + jj) * a.ldc;
                if (EPI == EPI_STORE_T) {
                  a.C[o] = x;
                } else {
                  const __half h = __float2half_rn(x);
                  a.c_hi[o] = h;
                  a.c_lo[o] = __float2half_rn(x - __half2float(h));
                }
              }
          }
          continue;
        }
        if (EPI == EPI_KV_SPLIT) {
          // [2i d, 2i d + d) -> K_i, [2i d + d, 2(i+1) d) -> V_i^T, both as fp16
          // hi / lo of kv_scale * x for the attention GEMMs; V^T is written
          // straight from the row-per-lane registers (coalesced over rows).
          // With d % 32 == 0 a chunk lies wholly in one K or V block.
          const long long grow = (long long)ti.c_row + rbase + lane;
          const int layer = col0 / (2 * a.kv_d), w0 = col0 - layer * 2 * a.kv_d;
          if (a.kv_d % 32 == 0) {
            if (w0 >= a.kv_d) {
              if (lane < nrows) {
                __half *vh = a.vt_hi + ((long long)layer * a.kv_d + (w0 - a.kv_d)) * a.vt_ld + grow;
                __half *vl = a.vt_lo + ((long long)layer * a.kv_d + (w0 - a.kv_d)) * a.vt_ld + grow;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                  const float x = v[jj] * a.alpha * a.kv_scale;
                  range_check(x, a.range_flag);
                  const __half h = __float2half_rn(x);
                  vh[(long long)jj * a.vt_ld] = h;
                  vl[(long long)jj * a.vt_ld] = __float2half_rn(x - __half2float(h));
                }
              }
              continue;  // no K columns in this chunk
            }
          } else {
#pragma unroll 1
            for (int jj = 0; jj < 32; ++jj) {
              const int col = col0 + jj, ly = col / (2 * a.kv_d), w = col - ly * 2 * a.kv_d;
              if (col < N && w >= a.kv_d && lane < nrows) {
                const float x = v[jj] * a.alpha * a.kv_scale;
                range_check(x, a.range_flag);
                const __half h = __float2half_rn(x);
                const long long o = ((long long)ly * a.kv_d + (w - a.kv_d)) * a.vt_ld + grow;
                a.vt_hi[o] = h;
                a.vt_lo[o] = __float2half_rn(x - __half2float(h));
              }
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) ebuf[lane * 33 + jj] = v[jj];
        __syncwarp();
        // lane -> (row lr of every 4, columns c4..c4+3): float4 global traffic,
        // 8 row groups per 32-column chunk
        const int lr = lane >> 3, c4 = (lane & 7) * 4;
        const int col = col0 + c4;
        const bool vec = col + 4 <= N && (a.ldc % 4) == 0 &&
                         (EPI != EPI_RESID && EPI != EPI_BIAS_RESID && EPI != EPI_BIAS_RESID_DUAL ||
         (a.ldr % 4) == 0) &&
                         (EPI != EPI_MULVEC && EPI != EPI_MULVEC_SPLIT || (a.vec_ld % 4) == 0) &&
                         (EPI != EPI_KV_SPLIT || (a.k_ld % 4) == 0);
        float4 bcol = make_float4(0.f, 0.f, 0.f, 0.f);
        if (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID ||
            EPI == EPI_BIAS_GELU_SPLIT || EPI == EPI_BIAS_RESID_DUAL || EPI == EPI_BIAS_DUAL) {
          bcol.x = col < N ? a.bias[col] : 0.f;
          bcol.y = col + 1 < N ? a.bias[col + 1] : 0.f;
          bcol.z = col + 2 < N ? a.bias[col + 2] : 0.f;
          bcol.w = col + 3 < N ? a.bias[col + 3] : 0.f;
        }
        // operands first (all loads in flight; C may alias R), then the stores
        float4 xo[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + lr;
          const long long grow = (long long)ti.c_row + rbase + rr;
          float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rr < nrows && col < N) {
            const float *src = nullptr;
            if (EPI == EPI_RESID || EPI == EPI_BIAS_RESID || EPI == EPI_BIAS_RESID_DUAL)
              src = a.R + grow * a.ldr + col;
            else if (EPI == EPI_MULVEC || EPI == EPI_MULVEC_SPLIT)
              src = a.vec + (long long)a.row_req[grow] * a.vec_ld + col;
            if (src) {
              if (vec) {
                o = *reinterpret_cast<const float4 *>(src);
              } else {
                o.x = src[0];
                if (col + 1 < N) o.y = src[1];
                if (col + 2 < N) o.z = src[2];
                if (col + 3 < N) o.w = src[3];
              }
            }
          }
          xo[it] = o;
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + lr;
          if (rr >= nrows || col >= N) continue;
          const long long grow = (long long)ti.c_row + rbase + rr;
          float x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = ebuf[rr * 33 + c4 + q] * a.alpha;
          const float ob[4] = {bcol.x, bcol.y, bcol.z, bcol.w};
          const float oo[4] = {xo[it].x, xo[it].y, xo[it].z, xo[it].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (EPI == EPI_BIAS) x[q] = x[q] + ob[q];
            else if (EPI == EPI_BIAS_DUAL) x[q] = x[q] + ob[q];
            else if (EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_GELU_SPLIT)
              x[q] = gelu_tanh_fast(x[q] + ob[q]);
            else if (EPI == EPI_RESID) x[q] = oo[q] + x[q];
            else if (EPI == EPI_BIAS_RESID || EPI == EPI_BIAS_RESID_DUAL)
              x[q] = oo[q] + (x[q] + ob[q]);
            else if (EPI == EPI_MULVEC || EPI == EPI_MULVEC_SPLIT) x[q] = oo[q] * x[q];
          }
          if (EPI == EPI_KV_SPLIT) {
            // K part of the layer (columns never straddle K / V for d % 4 == 0)
            const int layer = col / (2 * a.kv_d), w = col - layer * 2 * a.kv_d;
            if (w < a.kv_d) {
              const long long o = grow * a.k_ld + (long long)layer * a.kv_d + w;
              __half hq[4], lq[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float xs = x[q] * a.kv_scale;
                range_check(xs, a.range_flag);
                hq[q] = __float2half_rn(xs);
                lq[q] = __float2half_rn(xs - __half2float(hq[q]));
              }
              if (vec) {
                *reinterpret_cast<uint2 *>(a.k_hi + o) = *reinterpret_cast<const uint2 *>(hq);
                *reinterpret_cast<uint2 *>(a.k_lo + o) = *reinterpret_cast<const uint2 *>(lq);
              } else {
                for (int q = 0; q < 4 && col + q < N; ++q) {
                  a.k_hi[o + q] = hq[q];
                  a.k_lo[o + q] = lq[q];
                }
              }
            }
            continue;
          }
          if (EPI == EPI_STORE_SPLIT || EPI == EPI_BIAS_GELU_SPLIT || EPI == EPI_BIAS_RESID_DUAL ||
              EPI == EPI_BIAS_DUAL || EPI == EPI_MULVEC_SPLIT) {
            __half hq[4], lq[4];
            const float cs = a.c_scale != 0.f ? a.c_scale : 1.f;  // (power of two)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float xs = x[q] * cs;
              if (a.c_scale != 0.f) range_check(xs, a.range_flag);
              hq[q] = __float2half_rn(xs);
              lq[q] = __float2half_rn(xs - __half2float(hq[q]));
            }
            const long long o = grow * a.ldc + col;
            if (vec) {
              *reinterpret_cast<uint2 *>(a.c_hi + o) = *reinterpret_cast<const uint2 *>(hq);
              *reinterpret_cast<uint2 *>(a.c_lo + o) = *reinterpret_cast<const uint2 *>(lq);
            } else {
              for (int q = 0; q < 4 && col + q < N; ++q) {
                a.c_hi[o + q] = hq[q];
                a.c_lo[o + q] = lq[q];
              }
            }
            if (EPI != EPI_BIAS_RESID_DUAL && EPI != EPI_BIAS_DUAL) continue;
          }
          float *dst = a.C + grow * a.ldc + col;
          if (vec) {
            *reinterpret_cast<float4 *>(dst) = make_float4(x[0], x[1], x[2], x[3]);
          } else {
            for (int q = 0; q < 4 && col + q < N; ++q) dst[q] = x[q];
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          mbar_arrive_remote(cluster_addr(&acce[acc], 0));  // the leader's MMA waits on it
        else
          mbar_arrive(&acce[acc]);
      }
      ++j;
    }
  }
  if (warp == kEpiWarp0 && lane == 0) dbg_stamp(a.dbg, 6);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync_all();  // no CTA leaves while its peer's traffic targets it
  if (threadIdx.x == 0) dbg_stamp(a.dbg, 7);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps + launch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // resolved once (thread-safe static init); a driver entry point, not state
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D K-major map: inner dim = cols (K), outer = rows; box BK x box_rows;
// fp32 tiles land SWIZZLE_128B (one 128-B row), fp16 tiles SWIZZLE_64B
static int make_map(CUtensorMap *m, const void *base, bool f16, long long rows, long long cols,
                    long long ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_err(GR4AD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = f16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  f16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(GR4AD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GR4AD_OK;
}

static int num_sms() {
  // per device, queried once (this runs on every launch of the eager path)
  static int cached[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n;
  }
  return cached[dev];
}

template <int BN, int STAGES, bool BSPLIT, bool ASPLIT = false>
static int launch_tc(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbl,
                     const CUtensorMap &mal, const TcArgs &a, int epi, cudaStream_t st) {
  constexpr size_t stage = (size_t)BM * BK * 4 + (size_t)BN * BK * 4;  // (in-place splits)
  constexpr size_t smem = 1024 + STAGES * stage + 256 + kEpiWarps * 32 * 33 * sizeof(float);
  static_assert(smem <= 227 * 1024, "stage ring exceeds shared memory");
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int n_tiles = tiles_m * tiles_n * a.groups;
  const int grid = std::min(n_tiles, num_sms());
  const int cls = (a.mode == GM_PLAIN) ? KC_GEMM : KC_ATTN_GEMM;
#define GR_TC_EPI(E)                                                                          \
  case E: {                                                                                   \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(gemm_tc_kernel<BN, STAGES, E, BSPLIT, ASPLIT>),               \
                                 (int)smem));      \
    GR_LAUNCH(cls, st, gemm_tc_kernel<BN, STAGES, E, BSPLIT, ASPLIT>                           \
                       <<<grid, kTcThreads, smem, st>>>(ma, mb, mbl, mal, a, tiles_m, tiles_n,  \
                                                        n_tiles));                            \
    return GR4AD_OK;                                                                          \
  }
  if (epi == EPI_STORE_T || epi == EPI_STORE_T_SPLIT) {
    switch (epi) {
      GR_TC_EPI(EPI_STORE_T)
      GR_TC_EPI(EPI_STORE_T_SPLIT)
      default: break;
    }
  }
  if constexpr (BN == 64 && BSPLIT && ASPLIT) {  // few-row products (no 128-column LSE parts)
    switch (epi) {
      GR_TC_EPI(EPI_STORE)
      GR_TC_EPI(EPI_RESID)
      GR_TC_EPI(EPI_BIAS_RESID)
      GR_TC_EPI(EPI_BIAS_GELU_SPLIT)
      GR_TC_EPI(EPI_STORE_SPLIT)
      GR_TC_EPI(EPI_BIAS_RESID_DUAL)
      default: return set_err(GR4AD_ERR_UNSUPPORTED, "tc epilogue %d at BN=64", epi);
    }
  } else if constexpr (BN < 128) {
    return set_err(GR4AD_ERR_UNSUPPORTED, "tc epilogue %d at BN=%d", epi, BN);
  } else if constexpr (ASPLIT) {  // the head layers' dense products on pre-split activations
    switch (epi) {
      GR_TC_EPI(EPI_STORE)
      GR_TC_EPI(EPI_RESID)
      GR_TC_EPI(EPI_BIAS_RESID)
      GR_TC_EPI(EPI_BIAS_GELU_SPLIT)
      GR_TC_EPI(EPI_STORE_SPLIT)
      GR_TC_EPI(EPI_BIAS_RESID_DUAL)
      GR_TC_EPI(EPI_STORE_LSE)
      GR_TC_EPI(EPI_KV_SPLIT)
      GR_TC_EPI(EPI_MULVEC_SPLIT)
      default: return set_err(GR4AD_ERR_UNSUPPORTED, "pre-split-A tc epilogue %d", epi);
    }
  } else {
  switch (epi) {
    GR_TC_EPI(EPI_STORE)
    GR_TC_EPI(EPI_BIAS)
    GR_TC_EPI(EPI_BIAS_GELU)
    GR_TC_EPI(EPI_RESID)
    GR_TC_EPI(EPI_BIAS_RESID)
    GR_TC_EPI(EPI_MULVEC)
    GR_TC_EPI(EPI_KV_SPLIT)
    GR_TC_EPI(EPI_STORE_LSE)
    GR_TC_EPI(EPI_STORE_SPLIT)
    GR_TC_EPI(EPI_BIAS_DUAL)
    default: return set_err(GR4AD_ERR_UNSUPPORTED, "tc epilogue %d", epi);
  }
  }
#undef GR_TC_EPI
}

// CTA-pair launch (PAIR instantiation): 256 x BN tiles, clusters of two
template <int BN, int STAGES>
static int launch_tc_pair(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbl,
                          const CUtensorMap &mal, const TcArgs &a, int epi, cudaStream_t st) {
  constexpr size_t stage = (size_t)BM * BK * 4 + (size_t)BN * BK * 2;  // A hi + lo, half B hi + lo
  constexpr size_t smem = 1024 + STAGES * stage + 256 + kEpiWarps * 32 * 33 * sizeof(float);
  static_assert(smem <= 227 * 1024, "stage ring exceeds shared memory");
  const int tiles_m = (a.M + 2 * BM - 1) / (2 * BM), tiles_n = (a.N + BN - 1) / BN;
  const int n_tiles = tiles_m * tiles_n * a.groups;  // (per-request groups: GM_QK / GM_PV)
  const int grid = 2 * std::min(n_tiles, num_sms() / 2);
  const int cls = (a.mode == GM_PLAIN) ? KC_GEMM : KC_ATTN_GEMM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define GR_TC_PAIR(E)                                                                            \
  case E: {                                                                                      \
    auto *k = gemm_tc_kernel<BN, STAGES, E, true, true, true>;                                   \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(k), (int)smem));    \
    GR_LAUNCH(cls, st, GR_CUDA(cudaLaunchKernelEx(&cfg, k, ma, mb, mbl, mal, a, tiles_m,           \
                                                      tiles_n, n_tiles)));                       \
    return GR4AD_OK;                                                                             \
  }
  switch (epi) {
    GR_TC_PAIR(EPI_STORE)
    GR_TC_PAIR(EPI_RESID)
    GR_TC_PAIR(EPI_BIAS_RESID)
    GR_TC_PAIR(EPI_BIAS_GELU_SPLIT)
    GR_TC_PAIR(EPI_STORE_SPLIT)
    GR_TC_PAIR(EPI_BIAS_RESID_DUAL)
    GR_TC_PAIR(EPI_STORE_LSE)
    GR_TC_PAIR(EPI_KV_SPLIT)
    GR_TC_PAIR(EPI_MULVEC_SPLIT)
    default: return set_err(GR4AD_ERR_UNSUPPORTED, "pre-split-A tc epilogue %d", epi);
  }
#undef GR_TC_PAIR
}

// GR4AD_FEW_ROWS=0 keeps few-row products on the pair tiles (A/B aid)
static bool few_rows_enabled() {
  static const bool on = [] {
    const char *e = getenv("GR4AD_FEW_ROWS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// GR4AD_FEW_BN=64|128: tile width of the few-row products (A/B aid)
static int few_rows_bn() {
  static const int bn = [] {
    const char *e = getenv("GR4AD_FEW_BN");
    return e && atoi(e) == 128 ? 128 : 64;
  }();
  return bn;
}

// GR4AD_TC_PAIR=0 keeps the single-CTA kernel for every product (A/B aid)
static bool pair_enabled() {
  static const bool on = [] {
    const char *e = getenv("GR4AD_TC_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tc_eligible(long long lda, long long ldb, int K, const void *A, const void *B) {
  return (lda % 4 == 0) && (ldb % 4 == 0) && (K % 4 == 0) &&
         (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
}

long long *g_tc_dbg = nullptr;  // gr4ad_debug_tc_timeline
int g_dbg_few = 0;  // gr4ad_debug_tc_few_rows

int gemm_tc(const TcArgs &a_in, long long a_rows, long long a_cols, long long b_rows,
            long long b_cols, int epi, cudaStream_t st) {
  TcArgs a = a_in;
  if (g_tc_dbg) a.dbg = g_tc_dbg;
  if (g_dbg_few) a.few_rows = 1;
  if (a.M <= 0 || a.N <= 0 || a.groups <= 0) return GR4AD_OK;
  static const bool trace = getenv("GR4AD_TRACE") != nullptr;  // debug aid (read-only)
  if (trace)
    fprintf(stderr, "gemm_tc M=%d N=%d K=%d groups=%d mode=%d epi=%d lda=%lld ldb=%lld ldc=%lld "
                    "A=(%lld,%lld) B=(%lld,%lld) presplit=%d asplit=%d\n",
            a.M, a.N, a.K, a.groups, a.mode, epi, a.lda, a.ldb, a.ldc, a_rows, a_cols, b_rows,
            b_cols, a.b_hi != nullptr, a.a_hi != nullptr);
  prof_tag("tc M=%d N=%d K=%d g=%d mode=%d epi=%d A=%lldx%lld B=%lldx%lld split=%d%d few=%d", a.M,
           a.N, a.K, a.groups, a.mode, epi, a_rows, a_cols, b_rows, b_cols, a.a_hi != nullptr,
           a.b_hi != nullptr, a.few_rows);
  if (epi == EPI_KV_SPLIT && (!a.k_hi || !a.vt_hi))
    return set_err(GR4AD_ERR_UNSUPPORTED, "K|V^T split epilogue needs its fp16 outputs");
  const bool wide = a.N >= 256;
  const int box_n = wide ? 256 : 128;
  CUtensorMap ma, mb, mbl;
  if (a.a_hi) {  // both operands pre-split: TMA only, no on-chip conversion
    if (!a.b_hi || a.lda % 8 != 0 || a.ldb % 8 != 0)
      return set_err(GR4AD_ERR_UNSUPPORTED, "pre-split A needs pre-split B and 16-B fp16 rows");
    CUtensorMap mal;
    GR_TRY(make_map(&ma, a.a_hi, true, a_rows, a_cols, a.lda, BM));
    GR_TRY(make_map(&mal, a.a_lo, true, a_rows, a_cols, a.lda, BM));
    // (per-request groups of <= 128 rows would leave half of a pair tile empty)
    const bool pair_mode = a.mode == GM_PLAIN || ((a.mode == GM_QK || a.mode == GM_PV) && a.M > BM);
    // few rows per request (trunk, level 0): 128 x 128 single-CTA tiles --
    // twice the CTAs of 256 x 256 pairs at the same M, and a two-warp
    // epilogue per lane quarter; a choice by the rows' role, not the batch
    // size, so a request decodes bit-identically in any batch
    if (a.few_rows && a.mode == GM_PLAIN && few_rows_enabled()) {
      // 128 x 64 tiles where the epilogue allows (not the 128-column LSE parts)
      // and they still fit one wave (tile width does not change any element's
      // K order, so results are the same either way)
      const long long narrow_tiles = (long long)((a.M + BM - 1) / BM) * ((a.N + 63) / 64);
      const bool narrow = few_rows_bn() == 64 && epi != EPI_STORE_LSE && epi != EPI_KV_SPLIT &&
                          epi != EPI_MULVEC_SPLIT && narrow_tiles <= num_sms();
      const int bn = narrow ? 64 : 128;
      GR_TRY(make_map(&mb, a.b_hi, true, b_rows, b_cols, a.ldb, bn));
      GR_TRY(make_map(&mbl, a.b_lo, true, b_rows, b_cols, a.ldb, bn));
      if (narrow) return launch_tc<64, 8, true, true>(ma, mb, mbl, mal, a, epi, st);
      return launch_tc<128, 6, true, true>(ma, mb, mbl, mal, a, epi, st);
    }
    if (wide && pair_mode && pair_enabled()) {
      GR_TRY(make_map(&mb, a.b_hi, true, b_rows, b_cols, a.ldb, 128));
      GR_TRY(make_map(&mbl, a.b_lo, true, b_rows, b_cols, a.ldb, 128));
      return launch_tc_pair<256, 6>(ma, mb, mbl, mal, a, epi, st);
    }
    GR_TRY(make_map(&mb, a.b_hi, true, b_rows, b_cols, a.ldb, box_n));
    GR_TRY(make_map(&mbl, a.b_lo, true, b_rows, b_cols, a.ldb, box_n));
    return wide ? launch_tc<256, 4, true, true>(ma, mb, mbl, mal, a, epi, st)
                : launch_tc<128, 6, true, true>(ma, mb, mbl, mal, a, epi, st);
  }
  GR_TRY(make_map(&ma, a.A, false, a_rows, a_cols, a.lda, BM));
  if (a.b_hi) {
    if (a.ldb % 8 != 0) return set_err(GR4AD_ERR_UNSUPPORTED, "fp16 B rows need ldb %% 8 == 0");
    GR_TRY(make_map(&mb, a.b_hi, true, b_rows, b_cols, a.ldb, box_n));
    GR_TRY(make_map(&mbl, a.b_lo, true, b_rows, b_cols, a.ldb, box_n));
    return wide ? launch_tc<256, 4, true>(ma, mb, mbl, ma, a, epi, st)
                : launch_tc<128, 6, true>(ma, mb, mbl, ma, a, epi, st);
  }
  GR_TRY(make_map(&mb, a.B, false, b_rows, b_cols, a.ldb, box_n));
  return wide ? launch_tc<256, 4, false>(ma, mb, mb, ma, a, epi, st)
              : launch_tc<128, 6, false>(ma, mb, mb, ma, a, epi, st);
}

int gemm_tc_swapped(const TcArgs &a, long long a_rows, long long a_cols, long long b_rows,
                    long long b_cols, cudaStream_t st, int epi) {
  if (epi != EPI_STORE_T && epi != EPI_STORE_T_SPLIT)
    return set_err(GR4AD_ERR_UNSUPPORTED, "swapped tc gemm: epilogue %d", epi);
  if (a.M <= 0 || a.N <= 0 || a.groups <= 0) return GR4AD_OK;
  if (a.mode != GM_QK_T && a.mode != GM_PV_T)
    return set_err(GR4AD_ERR_UNSUPPORTED, "swapped tc gemm: mode %d", a.mode);
  static const bool trace = getenv("GR4AD_TRACE") != nullptr;  // debug aid (read-only)
  if (trace)
    fprintf(stderr, "gemm_tc M=%d N=%d K=%d groups=%d mode=%d epi=%d lda=%lld ldb=%lld ldc=%lld "
                    "A=(%lld,%lld) B=(%lld,%lld) presplit=%d asplit=%d swapped=1\n",
            a.M, a.N, a.K, a.groups, a.mode, epi, a.lda, a.ldb, a.ldc, a_rows, a_cols, b_rows,
            b_cols, a.b_hi != nullptr, a.a_hi != nullptr);
  prof_tag("tcT M=%d N=%d K=%d g=%d mode=%d epi=%d A=%lldx%lld B=%lldx%lld split=%d", a.M, a.N,
           a.K, a.groups, a.mode, epi, a_rows, a_cols, b_rows, b_cols, a.a_hi != nullptr);
  CUtensorMap ma, mal, mb;
  // N = beam rows per request: the smallest tile that holds them
  const int bn = a.N <= 32 ? 32 : (a.N <= 64 ? 64 : 128);
  GR_TRY(make_map(&mb, a.B, false, b_rows, b_cols, a.ldb, bn));
  if (a.a_hi) {
    if (a.lda % 8 != 0) return set_err(GR4AD_ERR_UNSUPPORTED, "fp16 A rows need lda %% 8 == 0");
    GR_TRY(make_map(&ma, a.a_hi, true, a_rows, a_cols, a.lda, BM));
    GR_TRY(make_map(&mal, a.a_lo, true, a_rows, a_cols, a.lda, BM));
    if (bn == 32) return launch_tc<32, 8, false, true>(ma, mb, mb, mal, a, epi, st);
    if (bn == 64) return launch_tc<64, 8, false, true>(ma, mb, mb, mal, a, epi, st);
    return launch_tc<128, 6, false, true>(ma, mb, mb, mal, a, epi, st);
  }
  GR_TRY(make_map(&ma, a.A, false, a_rows, a_cols, a.lda, BM));
  if (bn == 32) return launch_tc<32, 8, false, false>(ma, mb, mb, ma, a, epi, st);
  if (bn == 64) return launch_tc<64, 8, false, false>(ma, mb, mb, ma, a, epi, st);
  return launch_tc<128, 6, false, false>(ma, mb, mb, ma, a, epi, st);
}

}  // namespace gr

// debug aid (not part of the ABI header): every tcgen05 GEMM launch writes
// per-CTA %globaltimer stamps [CTA][8] into buf (NULL: off)
extern "C" void gr4ad_debug_tc_timeline(long long *buf) { gr::g_tc_dbg = buf; }
// debug aid: route every tcgen05 GEMM as a few-row product
extern "C" void gr4ad_debug_tc_few_rows(int on) { gr::g_dbg_few = on; }
