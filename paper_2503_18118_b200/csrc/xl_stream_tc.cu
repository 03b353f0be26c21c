// xl_stream_tc.cu -- K4b on the 5th-generation tensor cores: G = H^H H streamed
// from HBM (XLMIMO_MATERIALIZED), tcgen05.mma kind::tf32 with the accumulator in
// TMEM, operands staged by TMA (SWIZZLE_128B) through an mbarrier ring.
//
// Real-ified Gram: H is stored planar [drop][K][2][N] (rows = (user, re/im)), so
// the 2K x N row block of a drop is the K-major operand A, and R = A A^T (M = 128
// rows, rows >= 2K zero in shared memory; MMA N = 2K rounded up to 16) gives
//   Re G(i,j) = R(2i,2j) + R(2i+1,2j+1),   Im G(i,j) = R(2i,2j+1) - R(2i+1,2j).
// TF32 products of the RNA-pre-rounded H (K4a, tf32 = 1) accumulate in fp32 over
// a chunk of kChunk elements; chunk partials are combined in fp64 by
// gram_reduce_kernel (fp32 in-tile, fp64 across tiles).
//
// Persistent kernel, one CTA per SM, warp roles: warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer (one elected lane), warps 4..7 epilogue (TMEM lane
// quadrants 0..3), double-buffered TMEM accumulator so the epilogue of one chunk
// overlaps the MMAs of the next.  Bounded mbarrier waits trap instead of hanging.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <type_traits>
#include <type_traits>

#include "xl_common.cuh"

namespace {

constexpr int kStages = 12;
constexpr int kRows = 128;             // MMA M (rows >= 2K stay zero)
constexpr int kBoxK = 32;              // fp32 elements per row per stage (128 B, one swizzle atom)
constexpr int kStageBytes = kRows * kBoxK * 4;  // 16 KiB
constexpr int kChunk = 8192;           // elements per work item (one fp64 partial per item)
// The tensor core's fp32 accumulation truncates: each MMA leaves ~0.5 ulp of the running
// sum, a relative bias of ~3e-8 per MMA that grows with the run length (512 MMAs per
// accumulator left -2.5e-5 on the cfg4 diagonal = 1.2e-3 bit of ZF rate at K = 32).  So
// the TMEM accumulator restarts every kSubStages stages (4 MMAs each: <= 64 MMAs, bias
// <= ~3e-6); the epilogue folds the sub-chunk sums into a running fp32 sum kept in a third
// TMEM region (drain_subchunk) and writes the item's fp64 partial after the last one.
constexpr int kSubStages = 16;   // stream kernel (TF32): 16 stages x 4 MMAs (K = 8 each)
constexpr int kFSubStages = 8;   // fused kernel (fp16): 8 stages of 64 elements = 32 MMAs (K = 16 each)
constexpr int kPSubStages = 8;   // pair kernel: 8 stages x 4 MMAs (K = 100 rates: -4e-4 bit at 16)
constexpr int kThreads = 256;

// element blocks stacked per stage in the 128 MMA rows: 2K <= 32 -> 4 blocks, <= 64 -> 2, else 1
int rows_per_block(int K) { return 2 * K <= 32 ? 32 : 2 * K <= 64 ? 64 : 128; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

// Parity wait with a suspend-time hint: a waiting warp is parked (up to ~20 us per attempt,
// woken when the phase completes) instead of re-issuing try_wait, so waiting warps do not
// take issue slots from the working ones.  Bounded: a lost arrival traps instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done = 0;
  for (uint32_t it = 0; it < (1u << 20); ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(20000u)
        : "memory");
    if (done) return;
  }
  __trap();  // a lost arrival: abort the kernel rather than hang the GPU
}

__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap *map, void *dst, uint64_t *bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05): start >> 4,
// LBO = 16 B (unused for swizzled K-major), SBO = 1024 B (8 rows x 128 B),
// version 1 (bit 46), layout type 2 = SWIZZLE_128B (bits 61..63).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major (same fields as tf32_idesc)
__host__ __device__ constexpr uint32_t f16_idesc(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// one lane of a converged warp (elect.sync): the warp runs the issue loop together, so its
// descriptors and counters are warp-uniform and live in uniform registers, and one lane
// issues each tcgen05 instruction (no per-instruction R2UR / ELECT retry loop)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Epilogue of one TMEM sub-chunk (K <= 64 kernels).  `lane_base` = tmem + (32 q << 16), the
// thread's accumulator row at column acc_col, its running sum at run_col (same row, a third
// TMEM region).  Sub-chunks before the last fold the accumulator into the running sum in fp32
// (round to nearest: unbiased, unlike the tensor core's own accumulation); the last adds the
// running sum, pairs re/im rows with the neighbouring lane and writes
//   Re G(i,j) = R(2i,2j) + R(2i+1,2j+1),  Im G(i,j) = R(2i,2j+1) - R(2i+1,2j)
// (even lane: j-pairs 0..3 of each 16-column slab, odd lane: 4..7) into the item's fp64
// partial `out` (packed upper triangle).  16-column slabs keep the live set at 32 floats.
__device__ __forceinline__ void drain_subchunk(uint32_t lane_base, uint32_t acc_col, uint32_t run_col, int R, int K,
                                               int i, int plane, bool first, bool last, double *out,
                                               double post = 1.0, int j0 = 0) {
  for (int cb = 0; cb < (R + 15) / 16; ++cb) {
    float v[16];
    tmem_ld16(lane_base + acc_col + (uint32_t)(16 * cb), v);
    if (!first) {
      float r[16];
      tmem_ld16(lane_base + run_col + (uint32_t)(16 * cb), r);
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] += r[e];
    }
    if (!last) {
      tmem_st16(lane_base + run_col + (uint32_t)(16 * cb), v);
      continue;
    }
    float x[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] = __shfl_xor_sync(0xffffffffu, v[e], 1);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int jj = plane * 4 + h;
      const int j = j0 + 8 * cb + jj;
      float rr, rr2, ri, ir;  // R(2i,2j), R(2i+1,2j+1), R(2i,2j+1), R(2i+1,2j)
      if (plane == 0) { rr = v[2 * jj]; ri = v[2 * jj + 1]; ir = x[2 * jj]; rr2 = x[2 * jj + 1]; }
      else { rr = x[2 * jj]; ri = x[2 * jj + 1]; ir = v[2 * jj]; rr2 = v[2 * jj + 1]; }
      if (i < K && j < K && j >= i) {
        const int64_t p = (int64_t)i * K - (int64_t)i * (i - 1) / 2 + (j - i);
        out[2 * p] = ((double)rr + (double)rr2) * post;
        out[2 * p + 1] = (i == j) ? 0.0 : ((double)ri - (double)ir) * post;
      }
    }
  }
}

struct StreamParams {
  double *ws;        // partials [drop][chunk][blk][NP][2] (absolute drop index)
  int K;
  int rb;            // rows per element block in a stage (32, 64 or 128; >= 2K)
  int nblk;          // element blocks stacked in the 128 MMA rows (128 / rb)
  int n_mma;         // MMA N
  int64_t N;
  int n_chunks;      // per drop
  int64_t drop0;     // first drop of this batch
  int nb;            // drops in this batch
  uint32_t tmem_cols;
};

// stages of work item chunk c (chunk elements each): kb_per_chunk, fewer in the ragged last chunk
__device__ __forceinline__ int item_stages(int64_t N, int c, int kb_per_chunk, int spb, int chunk = kChunk) {
  const int64_t rem = N - (int64_t)c * chunk;
  const int64_t ns = (rem + spb - 1) / spb;
  return ns < kb_per_chunk ? (int)ns : kb_per_chunk;
}

__global__ void __launch_bounds__(kThreads, 1) gram_stream_tc_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                    StreamParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned stage ring
  uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *stages = base;
  uint64_t *full = (uint64_t *)(base + kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_base_sh = (uint32_t *)(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = P.K, R = 2 * K;
  const int64_t n_items = (int64_t)P.nb * P.n_chunks;

  // zero the ring once: rows >= 2K are never written by TMA and must read as 0
  for (int i = tid; i < kStages * kStageBytes / 16; i += kThreads) ((uint4 *)stages)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;
  const int kb_per_chunk = kChunk / (kBoxK * P.nblk);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int d = (int)(it / P.n_chunks), c = (int)(it - (int64_t)d * P.n_chunks);
        const int64_t x0 = (int64_t)c * kChunk;
        for (int kb = 0; kb < kb_per_chunk; ++kb) {
          const int64_t x = x0 + (int64_t)kb * kBoxK * P.nblk;
          if (x >= P.N) break;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], (uint32_t)(P.nblk * R * kBoxK * 4));
          // one contiguous 2K x 128 B tile per element block (tiled32 layout, N padded by K4a)
          const int64_t tile0 = (int64_t)d * (P.N / kBoxK) + x / kBoxK;
          for (int b = 0; b < P.nblk; ++b)
            tma_load_3d(&tmap, stages + stage * kStageBytes + b * P.rb * kBoxK * 4, &full[stage], 0, 0,
                        (int)(tile0 + b));
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = tf32_idesc(kRows, P.n_mma);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int d = (int)(it / P.n_chunks), c = (int)(it - (int64_t)d * P.n_chunks);
        (void)d;
        const int ns = item_stages(P.N, c, kb_per_chunk, kBoxK * P.nblk);
        for (int s0 = 0; s0 < ns; s0 += kSubStages, ++local) {  // one TMEM sub-chunk
          const int acc = local & 1;
          const uint32_t acc_phase = (local >> 1) & 1;
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t tmem_d = tmem + (uint32_t)(acc * P.n_mma);
          const int s1 = s0 + kSubStages < ns ? s0 + kSubStages : ns;
          for (int kb = s0; kb < s1; ++kb) {
            mbar_wait(&full[stage], phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(stages + stage * kStageBytes);
#pragma unroll
            for (int k = 0; k < kBoxK / 8; ++k) {  // 8 tf32 (32 B) per MMA along K
              const uint64_t desc = sw128_desc(sa + 32 * k);
              mma_tf32(tmem_d, desc, desc, idesc, (kb > s0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&empty[stage]);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[acc]);
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM lanes 32q..32q+31
    const int q = warp - 4;
    const int row = 32 * q + lane;
    const int blk = (32 * q) / P.rb;                 // element block of this quadrant
    const int lr = row - blk * P.rb;                 // row within the block
    const int i = lr >> 1, plane = lr & 1;
    const int col0 = blk * P.rb;                     // the block's diagonal columns
    const bool has_users = 32 * q - blk * P.rb < R;
    const int NP = K * (K + 1) / 2;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int d = (int)(it / P.n_chunks), c = (int)(it - (int64_t)d * P.n_chunks);
      double *out = P.ws + (((size_t)(P.drop0 + d) * P.n_chunks + c) * P.nblk + blk) * (size_t)(2 * NP);
      const int ns = item_stages(P.N, c, kb_per_chunk, kBoxK * P.nblk);
      for (int s0 = 0; s0 < ns; s0 += kSubStages, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tfull[acc], acc_phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (has_users)
          drain_subchunk(tmem + ((uint32_t)(32 * q) << 16), (uint32_t)(acc * P.n_mma + col0),
                         (uint32_t)(2 * P.n_mma + col0), R, K, i, plane, s0 == 0, s0 + kSubStages >= ns, out);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
  }
}

// ---------------------------------------------------------------------------
// Fused fp32 path (XLMIMO_FP32, XLMIMO_FUSED, K >= 9): the same tcgen05 TF32
// Gram, but the operand tiles are GENERATED into the swizzled shared-memory ring
// by 4 generator warps instead of being loaded by TMA -- H never touches HBM.
// Generator task = (user u, 4 consecutive elements): the fp64 anchor at the first
// element (distance, 1/r, phase reduced as frac(r/lambda) in fp64, north_star),
// then for the 4 elements an fp32 delta: Delta(r^2) = dd (2 dy + dd),
// delta = Delta / r_c^2, Delta r = r_c delta (1/2 - delta/8 + delta^2/16),
// phase = frac_c + Delta r / lambda (fp32, re-reduced), sin/cos by MUFU,
// amplitude a_c (1 + delta)^{-3/4} ~ a_c (1 - 3/4 delta + 21/32 delta^2); each
// row chunk of 4 TF32 (RNA) values is one 16-byte store.  Elements are taken in
// natural spatial order (the sum is order-free; no nested levels on this path).
// Launch constants of the fp16 task generator (kernel parameters: the constant bank, no
// registers).  A task's anchor is its centre: ey = (col + y_off) pitch, ez = (row + z_off)
// pitch with col/row the array indices of its first element.
struct GenConst {
  double pitch, inv_lambda;
  double y_off, z_off;  // (TE - 1)/2 - (n_cols - 1)/2, -(n_rows - 1)/2
  int64_t N, n_y;       // elements (ULA: the level's N), UPA row length
  double n_y_d, inv_ny;  // UPA: n_y and 1 / n_y as doubles
  int kind;
  float pitch_f, pl, cb0;  // pitch, 2 pi pitch / lambda, pitch pl / 2 (fp32)
};

inline GenConst make_gen_const(const xlh::ArrayP &a, int64_t N, int TE) {
  GenConst g;
  g.pitch = a.pitch;
  g.inv_lambda = 1.0 / a.lambda;
  g.kind = a.kind;
  g.N = N;
  g.n_y = a.n_y;
  g.n_y_d = (double)a.n_y;
  g.inv_ny = 1.0 / (double)a.n_y;
  const double n_cols = a.kind == XLMIMO_ULA ? (double)N : (double)a.n_y;
  g.y_off = 0.5 * (TE - 1) - 0.5 * (n_cols - 1.0);
  g.z_off = a.kind == XLMIMO_ULA ? 0.0 : -0.5 * ((double)a.n_z - 1.0);
  g.pitch_f = (float)a.pitch;
  g.pl = 6.28318530717958647692f * g.pitch_f * (float)g.inv_lambda;
  g.cb0 = 0.5f * g.pitch_f * g.pl;
  return g;
}

struct FusedParams {
  const double *pos;
  double *ws;        // partials [drop][chunk][NP][2]
  int K, kind;
  int64_t n_y, n_z, N;
  double lambda, pitch, sqrt_beta0;
  int rb, nblk;      // rows per element block, blocks stacked per stage (as StreamParams)
  int n_mma;
  int n_chunks;
  int chunk;         // elements per work item (a multiple of kChunk)
  int64_t n_drops;
  uint32_t tmem_cols;
  GenConst g;        // the generator's launch constants (TE of the instantiation)
  int u0, k_gen;     // users generated: u0 .. u0 + k_gen - 1 of the K (rows 2u, 2u + 1) ...
  int ka, b0;        // ... or, with b_row > 0, u0 .. u0 + ka - 1 then b0 .. b0 + k_gen - ka - 1
  int b_row;         // first stage row of the MMA's B operand: 0 (B = all rows) or 2 ka (cross)
  int n_acc;         // TMEM accumulators (2: double-buffered, 1 when 3 n_mma > 512)
};

// TF32 round-to-nearest, ties away from zero, as integer ALU work (sign-magnitude:
// add half a TF32 ulp to the magnitude, drop the 13 low mantissa bits) -- the same
// bits as cvt.rna.tf32.f32 for finite x, without its XU-pipe conversion.
__device__ __forceinline__ uint32_t tf32_rna(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

// byte offset of the 16-B chunk c (0..7) of row r in a SWIZZLE_128B K-major tile
__device__ __forceinline__ uint32_t sw128_off(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

constexpr int kTaskE = 8;          // elements per generator task (one fp64 anchor)

__device__ __forceinline__ void st_cs_v8(float *p, const uint32_t (&v)[8]) {  // 32-B aligned, evict-first
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void st_v8(float *p, const uint32_t (&v)[8]) {  // 32-B aligned, default (L2-resident)
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}



// The fused kernel's generator task: TE (8 or 16) consecutive elements t0 .. t0 + TE - 1 of
// one user, from an fp64 anchor at the task's CENTRE (element t0 + (TE - 1)/2, a half-
// integer position), so the Taylor offsets are |m'| <= (TE - 1)/2 pitches: a 16-element task
// has the truncation of gen_task_tf32's 8-element one (d^5/r^4 over 7.5 pitches) for half
// the anchors.  Same expansion as gen_task_tf32 with m' = m - (TE - 1)/2.  Output: the
// coefficients times 2^e (the drop's power-of-two scale, see gram_fused_tc_kernel) rounded
// to fp16 (round to nearest even: 11 significant bits, the precision of TF32) and packed
// in pairs, hr[q] = (re h_{2q}, re h_{2q+1}) low half first, hi likewise.  Full tasks
// (all TE elements < N) skip the per-element padding select.
// (double)t for 0 <= t < 2^52 without the XU-pipe I2F: t in the mantissa of 2^52, minus 2^52.
__device__ __forceinline__ double i2d_exact(int64_t t) {
  return __longlong_as_double(0x4330000000000000LL + t) - 4503599627370496.0;
}

// A generator's user: the fp64 geometry of xl::UserC and its amplitude sqrt(beta0) sqrt(x_eff)
// rounded to fp32 once per drop (the coefficient's amplitude is an fp32 product anyway).
struct __align__(16) GenUser {
  double xz2, y, z;
  float amp, unused;
};

// fp32 of a positive normal double whose exponent fits fp32 (truncated mantissa): the
// exponent field moves down by 1023 - 127 in modular 32-bit arithmetic (2 integer ops).
__device__ __forceinline__ float f64_trunc_f32(double x) {
  const uint32_t b = __funnelshift_l((uint32_t)__double2loint(x), (uint32_t)__double2hiint(x), 3);
  return __uint_as_float(b - (896u << 23));
}

// A GenUser from shared memory by its shared-window address (LDS, not generic loads).
__device__ __forceinline__ GenUser lds_user(uint32_t a) {
  GenUser g;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(g.xz2), "=d"(g.y) : "r"(a));
  asm volatile("ld.shared.f64 %0, [%1+16];" : "=d"(g.z) : "r"(a));
  asm volatile("ld.shared.f32 %0, [%1+24];" : "=f"(g.amp) : "r"(a));
  g.unused = 0.0f;
  return g;
}

// Anchor (task centre) of the task whose first element is t0, branch-free.  UPA tasks lie in
// one row (n_y % TE == 0): row = floor((t0 + 1/2) / n_y) in fp64 (all values < 2^53, exact
// after the +-1 fix-up), col = t0 - row n_y.
template <int KIND>
__device__ __forceinline__ void task_anchor(const GenConst &g, int64_t t0, double &ey, double &ez) {
  const double td = i2d_exact(t0);
  if constexpr (KIND == XLMIMO_ULA) {
    ey = (td + g.y_off) * g.pitch;
    ez = 0.0;
  } else {
    constexpr double kRnd = 6755399441055744.0;  // 1.5 2^52: x + kRnd - kRnd = rint(x)
    double row = (fma(td + 0.5, g.inv_ny, -0.5) + kRnd) - kRnd;
    double col = fma(-row, g.n_y_d, td);
    if (col < 0.0) { col += g.n_y_d; row -= 1.0; }
    if (col >= g.n_y_d) { col -= g.n_y_d; row += 1.0; }
    ey = (col + g.y_off) * g.pitch;
    ez = (row + g.z_off) * g.pitch;
  }
}

// One task's expansion about its centre (fm = m - (TE-1)/2, |fm| <= 7.5 for TE = 16):
//   phase fc + ca fm + cb fm^2 + cg fm^3 + cq fm^4, amplitude a0 + a1 fm + a2 fm^2.
struct TaskCoef {
  float fc, ca, cb, cg, cq, a0, a1, a2;
};

template <int KIND>
__device__ __forceinline__ TaskCoef task_coef(const GenUser &uc, double ey, double ez, const GenConst &g,
                                              float scale) {
  const double dy = ey - uc.y;
  double r2;
  if constexpr (KIND == XLMIMO_ULA) {
    r2 = fma(dy, dy, uc.xz2);
  } else {
    const double dz = ez - uc.z;
    r2 = fma(dy, dy, fma(dz, dz, uc.xz2));
  }
  // 1/r: MUFU seed + one Newton step (relative error ~3e-13: ~5e-7 rad of phase at 10^5
  // wavelengths, far below the fp16 operand's 2^-11)
  const double ir = xl::rsqrt_newton(r2);
  const double qc = (r2 * ir) * g.inv_lambda;
  constexpr double kRnd = 6755399441055744.0;  // qc - rint(qc) on the FP64 pipe (|qc| < 2^51)
  const double qf = qc - ((qc + kRnd) - kRnd);
  constexpr float k2pi = 6.28318530717958647692f;
  TaskCoef c;
  // fp64 -> fp32 without the XU-pipe F2F: qf + 1.5 and u + 3 lie in [1, 2] and [2, 4] (fixed
  // binade, + half a float ulp so the truncation rounds), 1/r is a normal float
  c.fc = fmaf(f64_trunc_f32(qf + (1.5 + 0x1p-24)), k2pi, -1.5f * k2pi);
  const float irf = f64_trunc_f32(ir);
  const float u = f64_trunc_f32(fma(dy, ir, 3.0 + 0x1p-23)) - 3.0f;
  const float w = fmaf(-u, u, 1.0f) * irf;  // (1 - u^2) / r
  const float p1 = g.pitch_f * irf;           // pitch / r
  // pl = 2 pi pitch / lambda, pp = pitch pl:
  //   ca = u pl, cb = w pp / 2, cg = -u w p1 pp / 2, cq = w (5u^2 - 1) p1^2 pp / 8
  c.ca = u * g.pl;
  c.cb = w * g.cb0;
  c.cg = -u * p1 * c.cb;
  c.cq = 0.25f * c.cb * fmaf(5.0f * u, u, -1.0f) * (p1 * p1);
  float sq;  // r^{-1/2} from the fp32 1/r (one MUFU, no second double -> float conversion)
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(irf));  // irf >= 2^-126: no denormal path
  // amplitude ac (1 + a1' fm + a2' fm^2): a1' = -3/2 u p1, a2' = 15/8 u^2 p1^2 - 3/4 w p1 pitch
  const float ac = uc.amp * irf * sq * scale;
  c.a0 = ac;
  const float acp = ac * p1;
  c.a1 = acp * (-1.5f * u);
  c.a2 = acp * fmaf(1.875f * u, u * p1, -0.75f * w * g.pitch_f);
  return c;
}

// h_m = a(fm) e^{-j phase(fm)} for the TE elements, times the drop scale (in a0..a2), rounded
// to fp16 (round to nearest even: 11 significant bits, the precision of TF32) and packed in
// pairs, hr[q] = (re h_{2q}, re h_{2q+1}) low half first, hi likewise.  Elements m and
// TE-1-m sit at fm = +-f: the even part of the phase E = fc + cb f^2 + cq f^4, the odd slope
// O = ca + cg f^2 and the even amplitude A = a0 + a2 f^2 are shared, ph = E +- f O,
// a = A +- f a1 (2.5 + 1.5 FFMA per element instead of the 4 + 2 of two Horner chains).
template <int TE>
__device__ __forceinline__ void task_emit(const TaskCoef &c, uint32_t (&hr)[TE / 2], uint32_t (&hi)[TE / 2]) {
  float re[TE], im[TE];
#pragma unroll
  for (int j = 0; j < TE / 2; ++j) {
    const float f = (float)j + 0.5f;  // |m - kMid| of the pair (TE/2 - 1 - j, TE/2 + j)
    const float f2 = f * f;
    const float E = fmaf(fmaf(c.cq, f2, c.cb), f2, c.fc);
    const float O = fmaf(c.cg, f2, c.ca);
    const float A = fmaf(c.a2, f2, c.a0);
    const int mp = TE / 2 + j, mn = TE / 2 - 1 - j;
    float sp, cp, sn, cn;
    __sincosf(fmaf(f, O, E), &sp, &cp);
    __sincosf(fmaf(-f, O, E), &sn, &cn);
    const float ap = fmaf(f, c.a1, A), an = fmaf(-f, c.a1, A);
    re[mp] = ap * cp;
    im[mp] = -ap * sp;
    re[mn] = an * cn;
    im[mn] = -an * sn;
  }
#pragma unroll
  for (int m = 0; m < TE / 2; ++m) {
    const __half2 hre = __floats2half2_rn(re[2 * m], re[2 * m + 1]);
    const __half2 him = __floats2half2_rn(im[2 * m], im[2 * m + 1]);
    hr[m] = *reinterpret_cast<const uint32_t *>(&hre);
    hi[m] = *reinterpret_cast<const uint32_t *>(&him);
  }
}

// Zero the elements m >= nv (past the array's end; only the array's last task has nv < TE).
template <int TE>
__device__ __forceinline__ void task_pad(int nv, uint32_t (&hr)[TE / 2], uint32_t (&hi)[TE / 2]) {
#pragma unroll
  for (int m = 0; m < TE; ++m)
    if (m >= nv) {
      const uint32_t keep = (m & 1) ? 0x0000FFFFu : 0xFFFF0000u;
      hr[m >> 1] &= keep;
      hi[m >> 1] &= keep;
    }
}

// One whole task: anchor at t0 (first element), nv = elements inside the array.
template <int TE, int KIND>
__device__ __forceinline__ void gen_task_h(const GenUser &uc, int64_t t0, int nv, const GenConst &g, float scale,
                                           uint32_t (&hr)[TE / 2], uint32_t (&hi)[TE / 2]) {
  double ey, ez;
  task_anchor<KIND>(g, t0, ey, ez);
  task_emit<TE>(task_coef<KIND>(uc, ey, ez, g, scale), hr, hi);
  if (nv < TE) task_pad<TE>(nv, hr, hi);
}

// The same expansion with fp32 outputs rounded to TF32 (round to nearest, ties away:
// tf32_rna) for the TF32 kernels, element m = 0..TE-1 in vr[m], vi[m]; elements m >= nv
// (past the array's end) are 0.
template <int TE>
__device__ __forceinline__ void task_emit_tf32(const TaskCoef &c, int nv, uint32_t (&vr)[TE], uint32_t (&vi)[TE]) {
#pragma unroll
  for (int j = 0; j < TE / 2; ++j) {
    const float f = (float)j + 0.5f;
    const float f2 = f * f;
    const float E = fmaf(fmaf(c.cq, f2, c.cb), f2, c.fc);
    const float O = fmaf(c.cg, f2, c.ca);
    const float A = fmaf(c.a2, f2, c.a0);
    const int mp = TE / 2 + j, mn = TE / 2 - 1 - j;
    float sp, cp, sn, cn;
    __sincosf(fmaf(f, O, E), &sp, &cp);
    __sincosf(fmaf(-f, O, E), &sn, &cn);
    const float ap = mp < nv ? fmaf(f, c.a1, A) : 0.0f;
    const float an = mn < nv ? fmaf(-f, c.a1, A) : 0.0f;
    vr[mp] = tf32_rna(ap * cp);
    vi[mp] = tf32_rna(-ap * sp);
    vr[mn] = tf32_rna(an * cn);
    vi[mn] = tf32_rna(-an * sn);
  }
}

template <int TE, int KIND>
__device__ __forceinline__ void gen_task_tf32(const GenUser &uc, int64_t t0, int nv, const GenConst &g,
                                              uint32_t (&vr)[TE], uint32_t (&vi)[TE]) {
  double ey, ez;
  task_anchor<KIND>(g, t0, ey, ez);
  task_emit_tf32<TE>(task_coef<KIND>(uc, ey, ez, g, 1.0f), nv, vr, vi);
}

constexpr int kGenWarps = 2;       // pair kernels: warps per generator group (arrivals per full barrier)
constexpr int kGenThreads = 32 * kGenWarps;
// Fused kernel (narrow stages, FCfg<false>): kFGroups groups of kFGenWarps warps; group g makes stages
// k = g (mod kFGroups) into ring slot k % kFStages.  The MMA consumes stages in order, so a
// group's next stage (k + groups) waits for slot k + groups - slots to be consumed; with
// parity waits are exact while groups <= slots.  Measured (148 cfg5 drops / 10^4 cfg3 /
// 10^3 cfg4, ms): 12 x 2 warps, 12 slots 9.82 / 2.78 / 2.35; 10 x 2, 12 slots 10.06 / 2.81 /
// 2.44; 5 x 4, 13 slots 10.69 / 2.96; 8 x 3 10.55; 4 x 6 12.82.
#ifndef XL_FGEN_WARPS
#define XL_FGEN_WARPS 2
#endif
#ifndef XL_FGEN_GROUPS
#define XL_FGEN_GROUPS 12
#endif
#ifndef XL_FSTAGES
#define XL_FSTAGES 12
#endif
constexpr int kFGenWarps = XL_FGEN_WARPS;
constexpr int kFGroups = XL_FGEN_GROUPS;
constexpr int kFStages = XL_FSTAGES;
constexpr int kEpiWarp0 = kFGenWarps * kFGroups;   // 24: warps 24..27 = TMEM lane quadrants 0..3
constexpr int kMmaWarp = kEpiWarp0 + 4;            // 28
constexpr int kFusedThreads = 32 * (kMmaWarp + 1);  // 928
static_assert(kEpiWarp0 % 4 == 0, "epilogue warp q must sit in TMEM lane quadrant q (warp % 4)");
static_assert(kFGroups <= kFStages, "a generator group may not lap a ring slot (parity waits)");

constexpr int kFBoxK = 64;  // fp16 elements per 128-B row of a fused stage (one swizzle atom)

// Stage shapes of gram_fused_tc_kernel: narrow (<= 64 users: 128 rows, 12 slots, 12 groups
// of 2 warps) and wide (<= 128 users: 256 rows, 6 slots of 32 KB, 6 groups of 4 warps; the
// MMA's A operand is the first 128 rows, its B operand all rows -- or, for a cross launch,
// the rows after them).  Same warps, threads and shared-memory budget.
template <bool WIDE>
struct FCfg {
  static constexpr int Groups = WIDE ? 6 : kFGroups, GenWarps = WIDE ? 4 : kFGenWarps;
  static constexpr int Stages = WIDE ? 6 : kFStages, Rows = WIDE ? 256 : kRows, MaxUsers = Rows / 2;
  static constexpr int GenThreads = 32 * GenWarps, StageBytes = Rows * 128, UBits = WIDE ? 7 : 6;
  // byte offset of su_all from the 1024-aligned base: stages, full/empty[Stages], tfull/tempty[2],
  // the TMEM base word (+16 B), rounded up to 64 B
  static constexpr int SuOff = (Stages * StageBytes + (2 * Stages + 4) * 8 + 16 + 63) & ~63;
  static_assert(GenWarps * Groups == kEpiWarp0 && Groups <= Stages, "FCfg warps / slots");
};

// Per-drop power-of-two scale of the fp16 operands: the largest coefficient magnitude of a
// user is sqrt(beta0) sqrt(x_eff) / x_eff^{3/2} = sqrt(beta0) / sqrt(xz2) (r >= x_eff), so
// 2^e with e = -ilogb(sqrt(beta0) / sqrt(min_u xz2)) puts the drop's largest |h| in [1, 2)
// and keeps the rest of it far inside fp16's normal range; the Gram is scaled by 4^e, undone
// exactly in the epilogue.  Generators (from su) and epilogue (from pos via make_user)
// evaluate the same doubles, so both sides use the same e.
__device__ __forceinline__ float scale_of_min_xz2(double min_xz2, double sqrt_beta0) {
  const int e = -ilogb(sqrt_beta0 / sqrt(min_xz2));
  return __int_as_float((127 + e) << 23);
}
__device__ __forceinline__ float drop_scale(const GenUser *su, int K, double sqrt_beta0) {
  double m = su[0].xz2;
  for (int u = 1; u < K; ++u) m = fmin(m, su[u].xz2);
  return scale_of_min_xz2(m, sqrt_beta0);
}
__device__ __forceinline__ float epi_drop_scale(const double *pos, int K, int kind, double sqrt_beta0, int lane,
                                                int ka = 1 << 30, int boff = 0) {
  double m = INFINITY;  // users 0 .. ka - 1, then ka + boff ..: the generators' users
  for (int u = lane; u < K; u += 32)
    m = fmin(m, xl::make_user(pos + (u < ka ? u : u + boff) * 3, kind, sqrt_beta0).xz2);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  return scale_of_min_xz2(m, sqrt_beta0);
}

template <int TE, int KIND, bool WIDE>
__global__ void __launch_bounds__(kFusedThreads, 1) gram_fused_tc_kernel(FusedParams P) {
  using C = FCfg<WIDE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *stages = base;
  uint64_t *full = (uint64_t *)(base + C::Stages * C::StageBytes);
  uint64_t *empty = full + C::Stages;
  uint64_t *tfull = empty + C::Stages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_base_sh = (uint32_t *)(tempty + 2);
  GenUser *su_all = (GenUser *)(base + C::SuOff);  // [groups][MaxUsers], past the TMEM base word

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = P.K, KG = P.k_gen, R = 2 * KG;  // K: the drop's users (indexing), KG: generated here
  const int64_t n_items = P.n_drops * P.n_chunks;
  for (int i = tid; i < C::Stages * C::StageBytes / 16; i += kFusedThreads)
    ((uint4 *)stages)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < C::Stages; ++s) {
      mbar_init(&full[s], C::GenWarps);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;
  const int kb_per_chunk = P.chunk / (kFBoxK * P.nblk);

  if (warp < kEpiWarp0) {  // ---------------- generators: group g makes stages k = g (mod 8)
    // The global stage sequence k (the MMA issuer's order) lives in slot k % 12 with
    // phase (k / 12) & 1; 12 slots for 8 groups let a group start its next stage
    // while the MMA still holds its previous one.
    const int grp = warp / C::GenWarps, gtid = tid - grp * C::GenThreads;
    GenUser *su = su_all + grp * C::MaxUsers;
    // the same address in the shared window, from the (constant) window offset of smem_raw
    uint32_t su_s = ((smem_u32(smem_raw) + 1023u) & ~1023u) + (uint32_t)C::SuOff + (uint32_t)(grp * C::MaxUsers) * 32u;
    asm volatile("" : "+r"(su_s));  // opaque: kept in a register, not re-derived per task
    // element blocks stacked in the 128 rows (as in the stream kernel): block b of a
    // stage covers elements xs + 64 b .. + 63 (fp16: 64 per 128-B row) in rows rb*b .. rb*b + 2K - 1
    constexpr int kTpr = kFBoxK / TE;      // tasks per user row of a block (4 or 8)
    const int n_tasks = P.nblk * KG * kTpr;
    constexpr int kUStep = C::GenThreads / kTpr;  // users a thread's task advances by
    static_assert(C::GenThreads % kTpr == 0, "task stepping assumes kTpr | GenThreads");
    const int g8 = gtid % kTpr;
    // The thread's tasks of a stage (the same every stage): task = (blk, u, g8) with
    // task = blk tpb + u kTpr + g8 for task = gtid, gtid + kFGenThreads, ...; the stride is a
    // multiple of kTpr, so g8 is the thread's constant.  Byte j of tdesc = u | blk << UBits of
    // its j-th task; n_my <= n_tasks / GenThreads <= 4 (TE = 16) or 8 (TE = 8) since nblk KG <=
    // MaxUsers (wide: nblk = 1, u < 128).
    using Desc = typename std::conditional<kTpr <= 4, uint32_t, uint64_t>::type;  // n_my <= kTpr bytes
    Desc tdesc = 0;
    int n_my = 0;
    {
      int u = gtid / kTpr, blk = 0;
      while (u >= KG) { u -= KG; ++blk; }
      for (int task = gtid; task < n_tasks; task += C::GenThreads, ++n_my) {
        tdesc |= (Desc)(u | (blk << C::UBits)) << (8 * n_my);
        u += kUStep;
        while (u >= KG) { u -= KG; ++blk; }
      }
    }
    const uint32_t code0 = (uint32_t)tdesc & 0xFFu;
    const Desc rest0 = tdesc >> 8;
    const uint32_t stages_base = smem_u32(stages);
    int64_t kstart = 0;  // global index of the item's first stage
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / P.n_chunks;
      const int c = (int)(it - d * P.n_chunks);
      const int64_t x0 = (int64_t)c * P.chunk;
      const int64_t rem = P.N - x0;
      const int spb = kFBoxK * P.nblk;  // elements per stage
      const int ns = (int)(((rem < P.chunk ? rem : P.chunk) + spb - 1) / spb);
      int64_t k = kstart + (((int64_t)grp - kstart) % C::Groups + C::Groups) % C::Groups;
      kstart += ns;
      if (k >= kstart) continue;  // no stage of this item for this group
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(C::GenThreads) : "memory");
      for (int u = gtid; u < KG; u += C::GenThreads) {
        const double *p = P.pos + (d * K + (u < P.ka ? P.u0 + u : P.b0 + (u - P.ka))) * 3;
        const xl::UserC uc = xl::make_user(p, P.kind, P.sqrt_beta0);
        su[u] = GenUser{uc.xz2, uc.y, uc.z, (float)uc.amp, 0.0f};
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(C::GenThreads) : "memory");
      const float scale = drop_scale(su, KG, P.sqrt_beta0);
      // A task = (blk, u, g8) with task = blk tpb + u kTpr + g8; the stride kFGenThreads is a
      // multiple of kTpr, so g8 is the thread's constant and u steps by kUStep.  Software
      // pipeline: the next task's anchor and coefficients (the serial fp64 chain) are formed in
      // the same basic block as the current task's phasors, so the chain's latency hides
      // behind the MUFU work; the next task of a stage's last one is the first of the group's
      // next stage.
      auto prep = [&](int64_t xs_, uint32_t code, TaskCoef &c_, int &nv_, int &row0_) {
        const int u_ = (int)(code & ((1u << C::UBits) - 1u)), blk_ = (int)(code >> C::UBits);
        const int64_t t0 = xs_ + (kFBoxK * blk_ + TE * g8);
        double ey, ez;
        task_anchor<KIND>(P.g, t0, ey, ez);
        c_ = task_coef<KIND>(lds_user(su_s + 32u * (uint32_t)u_), ey, ez, P.g, scale);
        const int64_t left = P.N - t0;
        nv_ = left < TE ? (int)left : TE;
        row0_ = blk_ * P.rb + 2 * u_;
      };
      int64_t xs = x0 + (k - (kstart - ns)) * spb;
      TaskCoef tc;
      int nv, row0;
      prep(xs, code0, tc, nv, row0);
      for (; k < kstart; k += C::Groups) {
        const int slot = (int)(k % C::Stages);
        const uint32_t slot_base = stages_base + slot * C::StageBytes;
        mbar_wait(&empty[slot], ((uint32_t)(k / C::Stages) & 1) ^ 1);
        Desc rest = rest0;  // codes of the tasks after the current one
        for (int j = n_my; j > 0; --j) {
          const bool last = j == 1;  // the next task is the first of the group's next stage
          const uint32_t code_n = last ? code0 : (uint32_t)rest & 0xFFu;
          rest >>= 8;
          const int64_t xsn = last ? xs + (int64_t)C::Groups * spb : xs;
          TaskCoef cn;
          int nvn, rown;
          prep(xsn, code_n, cn, nvn, rown);
          uint32_t hr[TE / 2], hi[TE / 2];
#ifdef XL_EXP_NO_GEN  // tuning experiment: the MMA / epilogue-bound rate (results invalid)
#pragma unroll
          for (int m = 0; m < TE / 2; ++m) hr[m] = hi[m] = (uint32_t)(xs + m);
#else
          task_emit<TE>(tc, hr, hi);
          if (nv < TE) task_pad<TE>(nv, hr, hi);
#endif
          // SWIZZLE_128B: 16-B chunk c of row r at r 128 + ((c ^ (r & 7)) << 4); row0 is even, so
          // the Im row's key is (row0 & 7) ^ 1, and the task's chunks are c0, c0 ^ 1 (c0 even)
          const uint32_t rbase = slot_base + (uint32_t)row0 * 128u;
          const uint32_t key = (uint32_t)((TE / 8) * g8) ^ (uint32_t)(row0 & 7);
#pragma unroll
          for (int h = 0; h < TE / 8; ++h) {  // 8 fp16 = one 16-B chunk of the 128-B row
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((key ^ (uint32_t)h) << 4)),
                         "r"(hr[4 * h]), "r"(hr[4 * h + 1]), "r"(hr[4 * h + 2]), "r"(hr[4 * h + 3])
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};"
                         ::"r"(rbase + 128u + ((key ^ 1u ^ (uint32_t)h) << 4)),
                         "r"(hi[4 * h]), "r"(hi[4 * h + 1]), "r"(hi[4 * h + 2]), "r"(hi[4 * h + 3])
                         : "memory");
          }
          tc = cn;
          nv = nvn;
          row0 = rown;
          xs = xsn;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[slot]);  // GenWarps arrivals complete the stage
      }
    }
  } else if (warp == kMmaWarp) {  // ---------------- MMA issuer (whole warp, one elected lane issues)
    const uint32_t idesc = f16_idesc(kRows, P.n_mma);
    const uint64_t desc0 = sw128_desc(smem_u32(stages));  // slot s, k-step k: + s StageBytes/16 + 2k
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / P.n_chunks;
      const int c = (int)(it - d * P.n_chunks);
      const int ns = item_stages(P.N, c, kb_per_chunk, kFBoxK * P.nblk, P.chunk);
      for (int s0 = 0; s0 < ns; s0 += kFSubStages, ++local) {  // one TMEM sub-chunk
        const int acc = P.n_acc == 2 ? (local & 1) : 0;
        const uint32_t acc_phase = (P.n_acc == 2 ? (local >> 1) : local) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tmem_d = tmem + (uint32_t)(acc * P.n_mma);
        const int s1 = s0 + kFSubStages < ns ? s0 + kFSubStages : ns;
        for (int kb = s0; kb < s1; ++kb) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ds = desc0 + (uint64_t)(stage * (C::StageBytes >> 4));
          if (elect_one()) {
#ifdef XL_EXP_NO_MMA  // tuning experiment: the generator-bound rate (results invalid)
            mbar_arrive(&empty[stage]);
#else
#pragma unroll
            for (int k = 0; k < kFBoxK / 16; ++k)  // 16 fp16 (32 B) per MMA along K
              mma_f16(tmem_d, ds + 2 * k, ds + (uint64_t)(P.b_row * 8) + 2 * k, idesc, (kb > s0 || k > 0) ? 1u : 0u);
            mma_commit(&empty[stage]);
#endif
          }
          __syncwarp();
          if (++stage == C::Stages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {  // ---------------- epilogue, warps kEpiWarp0..+3 = TMEM lane quadrants 0..3
    const int q = warp - kEpiWarp0;
    const int row = 32 * q + lane;
    const int blk = (32 * q) / P.rb;
    const int lr = row - blk * P.rb;
    const int i = P.u0 + (lr >> 1), plane = lr & 1;  // the drop's user index of this row
    const int col0 = blk * P.rb;
    const bool cross = P.b_row > 0;  // rows = users u0.., columns = users b0..
    const bool has_users = 32 * q - blk * P.rb < (cross ? 2 * P.ka : R);
    const int n_cols = R - P.b_row, j0 = cross ? P.b0 : P.u0;
    const int NP = K * (K + 1) / 2;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / P.n_chunks;
      const int c = (int)(it - d * P.n_chunks);
      double *out = P.ws + (((size_t)d * P.n_chunks + c) * P.nblk + blk) * (size_t)(2 * NP);
      const float sc = epi_drop_scale(P.pos + (d * K + P.u0) * 3, KG, P.kind, P.sqrt_beta0, lane, P.ka,
                                      P.b0 - P.u0 - P.ka);
      const double post = 1.0 / ((double)sc * (double)sc);  // exact: sc is a power of two
      const int ns = item_stages(P.N, c, kb_per_chunk, kFBoxK * P.nblk, P.chunk);
      for (int s0 = 0; s0 < ns; s0 += kFSubStages, ++local) {
        const int acc = P.n_acc == 2 ? (local & 1) : 0;
        const uint32_t acc_phase = (P.n_acc == 2 ? (local >> 1) : local) & 1;
        mbar_wait(&tfull[acc], acc_phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (has_users)
          drain_subchunk(tmem + ((uint32_t)(32 * q) << 16), (uint32_t)(acc * P.n_mma + col0),
                         (uint32_t)(P.n_acc * P.n_mma + col0), n_cols, K, i, plane, s0 == 0, s0 + kFSubStages >= ns,
                         out, post, j0);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
  }
}

// ------------------------------------------------------------------ K > 64, fp32
// Fused fp32 Gram for 64 < K <= 1024 on tcgen05: the block-pair decomposition of the
// fp64 BLK kernel with the machinery above.  A work item is (drop, user-block pair
// bi <= bj, 8192-element chunk); a stage holds the A tile (block bi: 64 users x re/im =
// 128 rows x 32 elements) and, for bi < bj, the B tile (block bj) behind it in the same
// 32 KB slot; the MMA computes A B^T (M = N = 128, K = 8, four per stage) into a
// double-buffered TMEM accumulator, the epilogue writes the block's entries of the
// packed upper triangle of the (drop, chunk) partial (the fp64 combine over chunks is
// gram_reduce_rows_kernel).  Six 32 KB slots; su holds the pair's 128 users per group.
constexpr int kPSlots = 6;
constexpr int kPGroups = kPSlots;  // a group may not lap a slot: groups <= slots (parity waits)
constexpr int kPSlotBytes = 2 * kStageBytes;
constexpr int kPUsers = 64;
// Elements accumulated in fp32 TMEM per partial: the tensor core's fp32 accumulation
// drifts by ~6e-8 per MMA (1024 per 8192 elements: 1.1e-4 normalised at K = 1000,
// M = 35 000, over the fp32-tier tolerance), so the pair kernel closes a partial every
// 4096 elements (half the drift) and combines partials in fp64.
constexpr int kPChunk = 4096;

// the pair kernel's own warp layout: 6 generator groups of 2 warps, 4 epilogue warps,
// the MMA warp (no idle warps, so the register cap leaves the generators unspilled)
constexpr int kPEpiWarp0 = kPGroups * kGenWarps;    // 12
constexpr int kPMmaWarp = kPEpiWarp0 + 4;           // 16
constexpr int kPairThreads = 32 * (kPMmaWarp + 1);  // 544
struct FusedPairParams {
  const double *pos;
  double *ws;        // partials [drop][chunk][NP][2], NP = K(K+1)/2 over all K users
  int K, kind, nb, n_pairs;
  int64_t n_y, n_z, N;
  double lambda, pitch, sqrt_beta0;
  int n_chunks;
  int64_t n_drops;
  GenConst g;        // the generator's launch constants (TE = kTaskE)
};

// stages (32 elements each) of pair-kernel chunk c (kPChunk elements, fewer in the last)
__device__ __forceinline__ int pair_item_stages(int64_t N, int c) {
  const int64_t rem = N - (int64_t)c * kPChunk;
  const int64_t ns = (rem + kBoxK - 1) / kBoxK;
  return ns < kPChunk / kBoxK ? (int)ns : kPChunk / kBoxK;
}

__device__ __forceinline__ void pair_of(int pair, int nb, int &bi, int &bj) {
  bi = 0;
  while (pair >= nb - bi) { pair -= nb - bi; ++bi; }
  bj = bi + pair;
}

__global__ void __launch_bounds__(kPairThreads, 1) gram_fused_tc_pair_kernel(FusedPairParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *stages = base;
  uint64_t *full = (uint64_t *)(base + kPSlots * kPSlotBytes);
  uint64_t *empty = full + kPSlots;
  uint64_t *tfull = empty + kPSlots;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_base_sh = (uint32_t *)(tempty + 2);
  GenUser *su_all = (GenUser *)(((uintptr_t)(tmem_base_sh + 4) + 63) & ~(uintptr_t)63);  // [groups][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = P.K;
  const int64_t per_drop = (int64_t)P.n_pairs * P.n_chunks;
  const int64_t n_items = P.n_drops * per_drop;
  for (int i = tid; i < kPSlots * kPSlotBytes / 16; i += kPairThreads) ((uint4 *)stages)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < kPSlots; ++s) {
      mbar_init(&full[s], kGenWarps);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == kPMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;
  constexpr int kSpb = kBoxK;  // elements per stage

  if (warp < kPGroups * kGenWarps) {  // ---------------- generators: group g makes stages k = g (mod 6)
    // (6 groups for 6 slots of 32 KB: more groups could lap a slot and pass a parity wait
    // one phase early)
    const int grp = warp / kGenWarps, gtid = tid - grp * kGenThreads;
    GenUser *su = su_all + grp * (2 * kPUsers);
    const uint32_t stages_base = smem_u32(stages);
    int64_t kstart = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / per_drop;
      const int rem2 = (int)(it - d * per_drop);
      const int pair = rem2 / P.n_chunks, c = rem2 - pair * P.n_chunks;
      int bi, bj;
      pair_of(pair, P.nb, bi, bj);
      const bool diag = bi == bj;
      const int64_t x0 = (int64_t)c * kPChunk;
      const int64_t rem = P.N - x0;
      const int ns = (int)(((rem < kPChunk ? rem : kPChunk) + kSpb - 1) / kSpb);
      int64_t k = kstart + (((int64_t)grp - kstart) % kPGroups + kPGroups) % kPGroups;
      kstart += ns;
      if (k >= kstart) continue;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kGenThreads) : "memory");
      for (int u = gtid; u < 2 * kPUsers; u += kGenThreads) {
        const int gu = (u < kPUsers ? bi : bj) * kPUsers + (u & (kPUsers - 1));
        if (gu < K) {
          const xl::UserC uc = xl::make_user(P.pos + (d * K + gu) * 3, P.kind, P.sqrt_beta0);
          su[u] = GenUser{uc.xz2, uc.y, uc.z, (float)uc.amp, 0.0f};
        } else {
          su[u] = GenUser{1.0, 0.0, 0.0, 0.0f, 0.0f};  // padded user: amplitude 0
        }
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kGenThreads) : "memory");
      const int n_tasks = (diag ? kPUsers : 2 * kPUsers) * (kBoxK / kTaskE);
      for (; k < kstart; k += kPGroups) {
        const int64_t xs = x0 + (k - (kstart - ns)) * kSpb;
        const int slot = (int)(k % kPSlots);
        const uint32_t slot_base = stages_base + slot * kPSlotBytes;
        mbar_wait(&empty[slot], ((uint32_t)(k / kPSlots) & 1) ^ 1);
        for (int task = gtid; task < n_tasks; task += kGenThreads) {
          const int u = task >> 2, g8 = task & 3;  // u < 64: A tile (rows 2u), else B tile (rows 128 + ...)
          const int row0 = 2 * u;
          const int64_t t0 = xs + kTaskE * g8;
          uint32_t vr[kTaskE], vi[kTaskE];
          const int64_t left = P.N - t0;
          const int nv = left < kTaskE ? (int)left : kTaskE;
          if (P.kind == XLMIMO_ULA) gen_task_tf32<kTaskE, XLMIMO_ULA>(su[u], t0, nv, P.g, vr, vi);
          else gen_task_tf32<kTaskE, XLMIMO_UPA>(su[u], t0, nv, P.g, vr, vi);
#pragma unroll
          for (int h = 0; h < kTaskE / 4; ++h) {
            const int chunk = (kTaskE / 4) * g8 + h;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(slot_base + sw128_off(row0, chunk)),
                         "r"(vr[4 * h]), "r"(vr[4 * h + 1]), "r"(vr[4 * h + 2]), "r"(vr[4 * h + 3])
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(slot_base + sw128_off(row0 + 1, chunk)),
                         "r"(vi[4 * h]), "r"(vi[4 * h + 1]), "r"(vi[4 * h + 2]), "r"(vi[4 * h + 3])
                         : "memory");
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[slot]);
      }
    }
  } else if (warp == kPMmaWarp) {  // ---------------- MMA issuer (whole warp, one elected lane issues)
    const uint32_t idesc = tf32_idesc(kRows, kRows);
    // (the original kernel's 12 slots over 8 groups satisfy the same groups <= slots rule)
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / per_drop;
      const int rem2 = (int)(it - d * per_drop);
      const int pair = rem2 / P.n_chunks, c = rem2 - pair * P.n_chunks;
      int bi, bj;
      pair_of(pair, P.nb, bi, bj);
      const bool diag = bi == bj;
      const int ns = pair_item_stages(P.N, c);
      for (int s0 = 0; s0 < ns; s0 += kPSubStages, ++local) {  // one TMEM sub-chunk (accumulation bias)
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tmem_d = tmem + (uint32_t)(acc * kRows);
        const int s1 = s0 + kPSubStages < ns ? s0 + kPSubStages : ns;
        for (int kb = s0; kb < s1; ++kb) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(stages + stage * kPSlotBytes);
          const uint32_t sb = diag ? sa : sa + kStageBytes;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBoxK / 8; ++kk)
              mma_tf32(tmem_d, sw128_desc(sa + 32 * kk), sw128_desc(sb + 32 * kk), idesc,
                       (kb > s0 || kk > 0) ? 1u : 0u);
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kPSlots) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (warp >= kPEpiWarp0) {  // ---------------- epilogue, warps kPEpiWarp0..+3 = TMEM lane quadrants
    const int q = warp - kPEpiWarp0;
    const int row = 32 * q + lane;
    const int il = row >> 1, plane = row & 1;
    const int64_t NP = (int64_t)K * (K + 1) / 2;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t d = it / per_drop;
      const int rem2 = (int)(it - d * per_drop);
      const int pair = rem2 / P.n_chunks, c = rem2 - pair * P.n_chunks;
      int bi, bj;
      pair_of(pair, P.nb, bi, bj);
      double *out = P.ws + ((size_t)d * P.n_chunks + c) * (size_t)(2 * NP);
      const int ns = pair_item_stages(P.N, c);
      for (int s0 = 0; s0 < ns; s0 += kPSubStages, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tfull[acc], acc_phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        drain_subchunk(tmem + ((uint32_t)(32 * q) << 16), (uint32_t)(acc * kRows), (uint32_t)(2 * kRows), kRows, K,
                       bi * kPUsers + il, plane, s0 == 0, s0 + kPSubStages >= ns, out, 1.0, bj * kPUsers);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (warp == kPMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// K4a for the tcgen05 stream: H of a batch of drops written straight into the tiled32
// TF32 layout [drop - drop0][N_pad / 32][2K][32] (row 2k = Re h_k, 2k + 1 = Im h_k) with
// the task generator above: a warp covers one 32-element tile for 8 users, lane =
// (user u = lane / 4, elements 8 (lane % 4) .. +7), so each lane stores 2 x 32 B and a
// warp writes sixteen full 128-B rows.  Block = 8 warps = 8 consecutive tiles; grid =
// (ceil(N_pad / 256), batch drops x ceil(K / 8) user groups).  Elements past N are 0.
template <int TE, int KIND>
__global__ void __launch_bounds__(256) h_materialise_tc_kernel(const double *pos, int K, int Kr, const GenConst g,
                                                               int64_t t_first, int64_t n_pad, double sqrt_beta0,
                                                               int64_t drop0, int n_ugrp, float *H, int l2_keep) {
  constexpr int LPR = 32 / TE, UPW = 32 / LPR;  // lanes per 32-element row, users per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bd = blockIdx.y / n_ugrp, ug = blockIdx.y - bd * n_ugrp;
  const int64_t tile = (int64_t)blockIdx.x * 8 + warp;
  if (tile * 32 >= n_pad) return;
  const int u = UPW * ug + lane / LPR, lt = lane % LPR;
  if (u >= Kr) return;
  float *row = H + (((size_t)bd * (n_pad / 32) + tile) * (2 * Kr) + 2 * u) * 32 + TE * lt;
  uint32_t vr[TE], vi[TE];
  if (u < K) {
    const xl::UserC c = xl::make_user(pos + ((drop0 + bd) * K + u) * 3, KIND, sqrt_beta0);
    const int64_t t0 = t_first + tile * 32 + TE * lt;
    const int64_t left = g.N - t0;
    gen_task_tf32<TE, KIND>(GenUser{c.xz2, c.y, c.z, (float)c.amp, 0.0f}, t0, left < TE ? (int)left : TE, g, vr,
                            vi);
  } else {  // padded user row (the pair stream reads whole 64-user blocks)
#pragma unroll
    for (int m = 0; m < TE; ++m) vr[m] = vi[m] = 0u;
  }
  // 256-bit stores (per plane TE / 8 of them, a lane's sectors whole): evict-first for the HBM
  // stream, default for an L2-sized chunk that is read back at once (the pair stream)
#pragma unroll
  for (int h = 0; h < TE / 8; ++h) {
    const uint32_t(&r8)[8] = *reinterpret_cast<const uint32_t(*)[8]>(vr + 8 * h);
    const uint32_t(&i8)[8] = *reinterpret_cast<const uint32_t(*)[8]>(vi + 8 * h);
    if (l2_keep) {
      st_v8(row + 8 * h, r8);
      st_v8(row + 32 + 8 * h, i8);
    } else {
      st_cs_v8(row + 8 * h, r8);
      st_cs_v8(row + 32 + 8 * h, i8);
    }
  }
}

// Per-drop power-of-two operand scale for the fp16 chunks (as the fused kernel's, R27):
// one warp per drop, min over users of xz2 (make_user), e = -ilogb(sqrt(beta0)/sqrt(min)).
__global__ void __launch_bounds__(256) drop_scale_kernel(const double *pos, int K, int kind, double sqrt_beta0,
                                                         int64_t n_drops, float *scale) {
  const int lane = threadIdx.x & 31;
  const int64_t d = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (d >= n_drops) return;
  scale[d] = epi_drop_scale(pos + d * K * 3, K, kind, sqrt_beta0, lane);
}

// K4a for the fp16 pair stream: H of a unit of drops x chunks in the tiled64 fp16 layout
// [drop - drop0][N_pad / 64][2 Kr][64] (row 2k = Re h_k, 2k + 1 = Im h_k; one 128-B swizzle
// row per user plane and tile), scaled per drop.  A warp covers one 64-element tile for
// 32 / (64 / TE) users; lane = (user, TE-element task), one 32-B (TE = 16) or 16-B store
// per plane.  Padded users (k >= K) and elements past N are 0.
template <int TE>
__global__ void __launch_bounds__(256) h_chunk_f16_kernel(const double *pos, int K, int Kr, const GenConst g,
                                                          int64_t t_first, int64_t n_pad, double sqrt_beta0,
                                                          int64_t drop0, int n_ugrp, const float *scale,
                                                          uint16_t *H) {
  constexpr int LPR = 64 / TE, UPW = 32 / LPR;  // lanes per user row, users per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bd = blockIdx.y / n_ugrp, ug = blockIdx.y - bd * n_ugrp;
  const int64_t tile = (int64_t)blockIdx.x * 8 + warp;
  if (tile * 64 >= n_pad) return;
  const int u = UPW * ug + lane / LPR, lt = lane % LPR;
  if (u >= Kr) return;
  uint16_t *row = H + (((size_t)bd * (n_pad / 64) + tile) * (2 * Kr) + 2 * u) * 64 + TE * lt;
  uint32_t hr[TE / 2], hi[TE / 2];
  if (u < K) {
    const xl::UserC c = xl::make_user(pos + ((drop0 + bd) * K + u) * 3, g.kind, sqrt_beta0);
    const GenUser uc{c.xz2, c.y, c.z, (float)c.amp, 0.0f};
    const int64_t t0 = t_first + tile * 64 + TE * lt;
    const int64_t left = g.N - t0;
    const int nv = left < TE ? (int)left : TE;
    if (g.kind == XLMIMO_ULA) gen_task_h<TE, XLMIMO_ULA>(uc, t0, nv, g, scale[drop0 + bd], hr, hi);
    else gen_task_h<TE, XLMIMO_UPA>(uc, t0, nv, g, scale[drop0 + bd], hr, hi);
  } else {
#pragma unroll
    for (int m = 0; m < TE / 2; ++m) hr[m] = hi[m] = 0u;
  }
#pragma unroll
  for (int h = 0; h < TE / 8; ++h) {  // L2-resident chunk: default-cached stores
    *reinterpret_cast<uint4 *>(row + 8 * h) = make_uint4(hr[4 * h], hr[4 * h + 1], hr[4 * h + 2], hr[4 * h + 3]);
    *reinterpret_cast<uint4 *>(row + 64 + 8 * h) =
        make_uint4(hi[4 * h], hi[4 * h + 1], hi[4 * h + 2], hi[4 * h + 3]);
  }
}

// K > 64 fp32 from a materialised chunk: the pair kernel's MMA and epilogue, fed by TMA
// from the tiled64 fp16 H of a unit of B drops x C element chunks (kPChunk each, L2-sized;
// fp16 operands with a per-drop scale as in the fused kernel, R27: half the L2 operand
// bytes of the round-1 TF32 chunks, which bound this kernel) instead of regenerating both
// 64-user blocks per pair.  tile index in the unit = (b * C + c) * (kPChunk / 64) + kb;
// rows of block b: [128 b, 128 b + 128); tcgen05.mma kind::f16, M = 128, N = 256.
constexpr int kSSlots = 4;                       // stream-pair ring: A 16 KB + B 32 KB per stage
constexpr int kSSlotBytes = 3 * kStageBytes;
struct StreamPairParams {
  double *ws;        // partials [drop][chunk][NP][2]
  int K, nb, n_pairs;
  int64_t N;
  int64_t drop0;     // first drop of the unit
  int n_ud, n_uc;    // drops and chunks in the unit
  int c0;            // first chunk of the unit
  int n_chunks;      // chunks per drop (partials layout)
  const float *scale;  // per-drop fp16 operand scale (absolute drop index)
};

__global__ void __launch_bounds__(256, 1) gram_stream_tc_pair_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                      StreamPairParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *stages = base;
  uint64_t *full = (uint64_t *)(base + kSSlots * kSSlotBytes);
  uint64_t *empty = full + kSSlots;
  uint64_t *tfull = empty + kSSlots;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_base_sh = (uint32_t *)(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = P.K;
  const int64_t per_drop = (int64_t)P.n_pairs * P.n_uc;
  const int64_t n_items = (int64_t)P.n_ud * per_drop;
  if (tid == 0) {
    for (int s = 0; s < kSSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_sh;
  constexpr int kTilesPerChunk = kPChunk / kFBoxK;  // fp16 tiles of 64 elements
  // item = (drop, block row bi, column blocks bj, bj + 1 (bj = bi + 2q), chunk): the B
  // operand is 256 rows (two 64-user blocks; rows past 2 K_pad come in as TMA zero fill)
  auto decode = [&](int64_t it, int &bl, int &bi, int &bj, int &cl) {
    bl = (int)(it / per_drop);
    const int rem = (int)(it - (int64_t)bl * per_drop);
    int w = rem / P.n_uc;
    cl = rem - w * P.n_uc;
    bi = 0;
    while (w >= (P.nb - bi + 1) / 2) { w -= (P.nb - bi + 1) / 2; ++bi; }
    bj = bi + 2 * w;
  };
  auto n_stages = [&](int cl) {
    const int64_t x0 = (int64_t)(P.c0 + cl) * kPChunk, rem = P.N - x0;
    return (int)(((rem < kPChunk ? rem : kPChunk) + kFBoxK - 1) / kFBoxK);
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int bl, bi, bj, cl;
        decode(it, bl, bi, bj, cl);
        const int ns = n_stages(cl);
        const int tile0 = (bl * P.n_uc + cl) * kTilesPerChunk;
        for (int kb = 0; kb < ns; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], (uint32_t)(3 * kStageBytes));
          uint8_t *dst = stages + stage * kSSlotBytes;
          tma_load_3d(&tmap, dst, &full[stage], 0, kRows * bi, tile0 + kb);
          tma_load_3d(&tmap, dst + kStageBytes, &full[stage], 0, kRows * bj, tile0 + kb);
          tma_load_3d(&tmap, dst + 2 * kStageBytes, &full[stage], 0, kRows * (bj + 1), tile0 + kb);
          if (++stage == kSSlots) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = f16_idesc(kRows, 2 * kRows);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++local) {
        int bl, bi, bj, cl;
        decode(it, bl, bi, bj, cl);
        const int ns = n_stages(cl);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tmem_d = tmem + (uint32_t)(acc * 2 * kRows);
        for (int kb = 0; kb < ns; ++kb) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(stages + stage * kSSlotBytes);
          const uint32_t sb = sa + kStageBytes;  // 256 rows: blocks bj, bj + 1
#pragma unroll
          for (int kk = 0; kk < kFBoxK / 16; ++kk)  // 16 fp16 (32 B) per MMA along K
            mma_f16(tmem_d, sw128_desc(sa + 32 * kk), sw128_desc(sb + 32 * kk), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[stage]);
          if (++stage == kSSlots) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue, warps 4..7 = TMEM lane quadrants
    const int q = warp - 4;
    const int row = 32 * q + lane;
    const int il = row >> 1, plane = row & 1;
    const int64_t NP = (int64_t)K * (K + 1) / 2;
    int local = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++local) {
      int bl, bi, bj, cl;
      decode(it, bl, bi, bj, cl);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      double *out = P.ws + ((size_t)(P.drop0 + bl) * P.n_chunks + (P.c0 + cl)) * (size_t)(2 * NP);
      const double sc = (double)P.scale[P.drop0 + bl];
      const double post = 1.0 / (sc * sc);  // exact: a power of two
      const int i = bi * kPUsers + il;
      for (int cb = 0; cb < 2 * kRows / 32; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 2 * kRows + 32 * cb), v);
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __shfl_xor_sync(0xffffffffu, v[e], 1);
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int jj = plane * 8 + h;
          const int jl = 16 * cb + jj;
          const int j = bj * kPUsers + jl;
          float rr, rr2, ri, ir;
          if (plane == 0) { rr = v[2 * jj]; ri = v[2 * jj + 1]; ir = x[2 * jj]; rr2 = x[2 * jj + 1]; }
          else { rr = x[2 * jj]; ri = x[2 * jj + 1]; ir = v[2 * jj]; rr2 = v[2 * jj + 1]; }
          if (i < K && j < K && j >= i) {
            const int64_t pp = (int64_t)i * K - (int64_t)i * (i - 1) / 2 + (j - i);
            out[2 * pp] = ((double)rr + (double)rr2) * post;
            out[2 * pp + 1] = (i == j) ? 0.0 : ((double)ri - (double)ir) * post;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

}  // namespace

namespace xlh {

bool stream_tc_supported(int K, int64_t N) { return K >= 9 && K <= 64 && (N % 4) == 0 && N >= kBoxK; }

int stream_tc_chunks(int64_t N) { return (int)((N + kChunk - 1) / kChunk); }

// Fused fp32 work items: the longest chunk (8192 .. 65536 elements, TMEM folding keeps the
// accumulation unbiased at any length) that still leaves >= 4 waves of items, so the fp64
// partials -- the kernel's only DRAM writes -- stay a small multiple of the output.
int fused_tc_chunk(int64_t N, int64_t n_drops) {
  int64_t c = kChunk;
  while (c < 65536 && n_drops * ((N + 2 * c - 1) / (2 * c)) >= 4 * 148) c *= 2;
  // the same number of items, of equal length (a ragged last item would idle its CTA's
  // generators): a multiple of 256 elements, whole stages for every block stacking
  const int64_t n = (N + c - 1) / c;
  const int64_t e = (N + n - 1) / n;
  return (int)((e + 255) / 256 * 256);
}
int fused_tc_chunks(int64_t N, int64_t n_drops) {
  const int c = fused_tc_chunk(N, n_drops);
  return (int)((N + c - 1) / c);
}

// UPA: a generator task (kTaskE consecutive elements off one fp64 anchor, the delta
// along y) must not cross a row of the n_y x n_z grid, so n_y must be a multiple of
// kTaskE; other UPAs take the CUDA-core fp32 kernel.
bool fused_tc_supported_geometry(const ArrayP &a) { return a.kind == XLMIMO_ULA || (a.n_y % kTaskE) == 0; }
bool fused_tc_supported(const ArrayP &a, int K) { return K >= 9 && K <= 64 && fused_tc_supported_geometry(a); }
// 64 < K <= kFusedTcMaxK on the fused kernel (wide, cross and narrow launches) unless XLMIMO_OPT_PAIR picks
// the block-pair kernel (1) or the TMA-fed pair stream (2)
bool fused_tc_wide_supported(const ArrayP &a, int K) {
  return K > 64 && K <= kFusedTcMaxK && fused_tc_supported_geometry(a);
}

// Fused fp32 Gram on tcgen05: partials [drop][chunk][block][NP][2] (NP = K(K+1)/2) into ws,
// fused_tc_chunks(N, n_drops) chunks per drop.  K <= 64: one narrow launch (element blocks
// stacked in the 128 rows for small K).  64 < K <= 128: a wide launch (rows = all K users,
// the MMA's A operand their first 64: the entries i < 64, j >= i) and a narrow one for users
// 64..K-1 (i, j >= 64), one element block each, writing disjoint entries of the same
// partials; every coefficient is generated once per launch that needs it (K + K - 64 user
// rows per element, against 4 x 64 for the block-pair kernel at K = 100).
int launch_fused_tc(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                    cudaStream_t s) {
  FusedParams P;
  P.pos = pos;
  P.ws = ws;
  P.K = K;
  P.kind = a.kind;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = N;
  P.lambda = a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  P.chunk = fused_tc_chunk(N, n_drops);
  P.n_chunks = fused_tc_chunks(N, n_drops);
  P.n_drops = n_drops;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = n_drops * P.n_chunks;
  const int grid = (int)(items < sms ? items : sms);
  // 16-element tasks wherever a task stays in one array row (every ULA; UPA rows of 16k)
  const bool te16 = a.kind == XLMIMO_ULA || a.n_y % 16 == 0;
  P.g = make_gen_const(a, N, te16 ? 16 : 8);
  auto launch = [&](int u0, int k_gen, bool wide, int b0 = 0, int kb = 0) {
    P.u0 = u0;
    P.k_gen = k_gen + kb;
    P.ka = k_gen;
    P.b0 = b0;
    P.b_row = kb > 0 ? 2 * k_gen : 0;
    if (wide || K > 64) {  // one element block per stage
      P.rb = wide ? 256 : kRows;
      P.nblk = 1;
      P.n_mma = (2 * (kb > 0 ? kb : k_gen) + 15) / 16 * 16;
    } else {
      P.rb = rows_per_block(K);
      P.nblk = kRows / P.rb;
      P.n_mma = P.nblk > 1 ? kRows : (2 * K + 15) / 16 * 16;
    }
    P.n_acc = 3 * P.n_mma <= 512 ? 2 : 1;  // accumulators + the running sum within 512 columns
    uint32_t cols = 32;
    while (cols < (uint32_t)((P.n_acc + 1) * P.n_mma)) cols <<= 1;
    P.tmem_cols = cols;
    auto run = [&](auto kern, int stage_bytes, int stages, int groups, int max_users) {
      const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 4) * 8 + 16 + 64 +
                          (size_t)groups * max_users * 32;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, kFusedThreads, smem, s>>>(P);
    };
    using CN = FCfg<false>;
    using CW = FCfg<true>;
    if (wide) {
      if (a.kind == XLMIMO_ULA) run(gram_fused_tc_kernel<16, XLMIMO_ULA, true>, CW::StageBytes, CW::Stages, CW::Groups, CW::MaxUsers);
      else if (te16) run(gram_fused_tc_kernel<16, XLMIMO_UPA, true>, CW::StageBytes, CW::Stages, CW::Groups, CW::MaxUsers);
      else run(gram_fused_tc_kernel<8, XLMIMO_UPA, true>, CW::StageBytes, CW::Stages, CW::Groups, CW::MaxUsers);
    } else {
      if (a.kind == XLMIMO_ULA) run(gram_fused_tc_kernel<16, XLMIMO_ULA, false>, CN::StageBytes, CN::Stages, CN::Groups, CN::MaxUsers);
      else if (te16) run(gram_fused_tc_kernel<16, XLMIMO_UPA, false>, CN::StageBytes, CN::Stages, CN::Groups, CN::MaxUsers);
      else run(gram_fused_tc_kernel<8, XLMIMO_UPA, false>, CN::StageBytes, CN::Stages, CN::Groups, CN::MaxUsers);
    }
    return check_launch("gram_fused_tc_kernel");
  };
  if (K <= 64) return launch(0, K, false);
  // rows in blocks of 64 users a0..: a wide launch over users a0 .. a0 + 127 (the block's
  // entries with j < a0 + 128) or a narrow one for the last block, then cross launches
  // (the block's 64 rows x 64 further users per launch) for the columns beyond
  for (int a0 = 0; a0 < K; a0 += 64) {
    const int rest = K - a0;
    int rc = rest <= 64 ? launch(a0, rest, false) : launch(a0, rest < 128 ? rest : 128, true);
    if (rc) return rc;
    for (int b0 = a0 + 128; b0 < K; b0 += 64) {
      rc = launch(a0, 64, true, b0, K - b0 < 64 ? K - b0 : 64);
      if (rc) return rc;
    }
  }
  return XLMIMO_OK;
}

// launches of launch_fused_tc for K users (the caller's launch counter)
int fused_tc_launches(int K) {
  if (K <= 64) return 1;
  int n = 0;
  for (int a0 = 0; a0 < K; a0 += 64) {
    ++n;
    for (int b0 = a0 + 128; b0 < K; b0 += 64) ++n;
  }
  return n;
}

int stream_tc_parts(int K) { return kRows / rows_per_block(K); }

// One batch: H in the tiled32 layout [nb][N/32][2K][32] fp32 (TF32-rounded, N a
// multiple of 128), partials for drops [drop0, drop0+nb).
// UPA rows must hold whole generator tasks (see fused_tc_supported).
bool materialise_tc_supported(const ArrayP &a) { return a.kind == XLMIMO_ULA || (a.n_y % kTaskE) == 0; }

int launch_h_materialise_tc(const ArrayP &a, const double *pos, int K, int64_t N, int64_t n_pad, int64_t drop0,
                            int nb, float *H, cudaStream_t s, int Kr, int64_t t_first, int l2_keep) {
  if (Kr < K) Kr = K;
  // 16-element tasks (16 users per warp) wherever a task stays in one array row
  const bool te16 = a.kind == XLMIMO_ULA || a.n_y % 16 == 0;
  const int upw = te16 ? 16 : 8;
  const int n_ugrp = (Kr + upw - 1) / upw;
  const dim3 grid((unsigned)((n_pad + 255) / 256), (unsigned)(nb * n_ugrp));
  const GenConst g = make_gen_const(a, N, te16 ? 16 : kTaskE);
  if (a.kind == XLMIMO_ULA)
    h_materialise_tc_kernel<16, XLMIMO_ULA><<<grid, 256, 0, s>>>(pos, K, Kr, g, t_first, n_pad, a.sqrt_beta0, drop0,
                                                                  n_ugrp, H, l2_keep);
  else if (te16)
    h_materialise_tc_kernel<16, XLMIMO_UPA><<<grid, 256, 0, s>>>(pos, K, Kr, g, t_first, n_pad, a.sqrt_beta0, drop0,
                                                                  n_ugrp, H, l2_keep);
  else
    h_materialise_tc_kernel<kTaskE, XLMIMO_UPA><<<grid, 256, 0, s>>>(pos, K, Kr, g, t_first, n_pad, a.sqrt_beta0,
                                                                      drop0, n_ugrp, H, l2_keep);
  return check_launch("h_materialise_tc_kernel");
}

int fused_tc_pair_chunks(int64_t N) { return (int)((N + kPChunk - 1) / kPChunk); }

// K > 64 fp32 from materialised chunks (gram_stream_tc_pair_kernel): units of B drops x
// C chunks with H (TF32, users padded to 64 nb) <= 112 MB so the pair reads hit L2.
struct PairUnit {
  int B, C;
  int Kp;
};
PairUnit stream_pair_unit(int K, int64_t n_drops, int64_t N) {
  PairUnit u;
  const int nb = (K + kPUsers - 1) / kPUsers;
  u.Kp = nb * kPUsers;
  const int64_t per = (int64_t)kPChunk * 2 * u.Kp * 2;  // one drop-chunk of H (fp16)
  const int64_t cap = 112ll << 20;  // most of the 126 MB L2 (measured best: 48 MB 84 ms, 112 MB 69 ms, 160+ MB 70 ms at E3)
  int64_t cells = cap / per;
  if (cells < 1) cells = 1;
  const int64_t chunks = fused_tc_pair_chunks(N);
  u.C = (int)(cells < chunks ? cells : chunks);
  int64_t b = cells / u.C;
  if (b > n_drops) b = n_drops;
  u.B = (int)(b < 1 ? 1 : b);
  return u;
}
size_t stream_pair_h_bytes(int K, int64_t n_drops, int64_t N) {  // H unit (fp16) + per-drop scales
  const PairUnit u = stream_pair_unit(K, n_drops, N);
  return ((size_t)u.B * u.C * kPChunk * 2 * u.Kp * 2 + 255) / 256 * 256 + (size_t)n_drops * sizeof(float);
}

int launch_stream_tc_pair(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                          float *Hbuf, cudaStream_t s) {
  auto enc = encode_fn();
  if (!enc) return set_error(XLMIMO_ECUDA, "stream_tc_pair: cuTensorMapEncodeTiled unavailable");
  const PairUnit u = stream_pair_unit(K, n_drops, N);
  uint16_t *H = reinterpret_cast<uint16_t *>(Hbuf);
  float *scale = reinterpret_cast<float *>(
      (char *)Hbuf + ((size_t)u.B * u.C * kPChunk * 2 * u.Kp * 2 + 255) / 256 * 256);
  const int nbk = u.Kp / kPUsers;
  const int chunks = fused_tc_pair_chunks(N);
  StreamPairParams P;
  P.ws = ws;
  P.K = K;
  P.nb = nbk;
  P.n_pairs = 0;  // items per (drop, chunk): block rows x column-block pairs
  for (int bi = 0; bi < nbk; ++bi) P.n_pairs += (nbk - bi + 1) / 2;
  P.N = N;
  P.n_chunks = chunks;
  P.scale = scale;
  {
    KTimer tm(s, "drop_scale");
    drop_scale_kernel<<<(unsigned)((n_drops + 7) / 8), 256, 0, s>>>(pos, K, a.kind, a.sqrt_beta0, n_drops, scale);
    tm.stop(s);
    count_launch();
  }
  const int te16 = a.kind == XLMIMO_ULA || a.n_y % 16 == 0;
  const size_t smem = 1024 + (size_t)kSSlots * kSSlotBytes + (2 * kSSlots + 4) * 8 + 16;
  cudaFuncSetAttribute(gram_stream_tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int64_t d0 = 0; d0 < n_drops; d0 += u.B) {
    const int nd = (int)((n_drops - d0) < u.B ? (n_drops - d0) : u.B);
    for (int c0 = 0; c0 < chunks; c0 += u.C) {
      const int ncu = (chunks - c0) < u.C ? chunks - c0 : u.C;
      const int64_t n_pad = (int64_t)ncu * kPChunk;
      {
        KTimer tm(s, "h_materialise");
        const int upw = te16 ? 8 : 4;
        const int n_ugrp = (u.Kp + upw - 1) / upw;
        const dim3 grid((unsigned)((n_pad + 511) / 512), (unsigned)(nd * n_ugrp));
        const GenConst g = make_gen_const(a, N, te16 ? 16 : 8);
        if (te16)
          h_chunk_f16_kernel<16><<<grid, 256, 0, s>>>(pos, K, u.Kp, g, (int64_t)c0 * kPChunk, n_pad, a.sqrt_beta0,
                                                      d0, n_ugrp, scale, H);
        else
          h_chunk_f16_kernel<8><<<grid, 256, 0, s>>>(pos, K, u.Kp, g, (int64_t)c0 * kPChunk, n_pad, a.sqrt_beta0,
                                                     d0, n_ugrp, scale, H);
        tm.stop(s);
        count_launch();
      }
      int rc = check_launch("h_chunk_f16_kernel");
      if (rc) return rc;
      CUtensorMap map;
      const cuuint64_t gdim[3] = {(cuuint64_t)kFBoxK, (cuuint64_t)(2 * u.Kp), (cuuint64_t)nd * (n_pad / kFBoxK)};
      const cuuint64_t gstride[2] = {(cuuint64_t)kFBoxK * 2, (cuuint64_t)kFBoxK * 2 * 2 * u.Kp};
      const cuuint32_t box[3] = {(cuuint32_t)kFBoxK, (cuuint32_t)kRows, 1};
      const cuuint32_t estride[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, (void *)H, gdim, gstride, box, estride,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return set_error(XLMIMO_ECUDA, "stream_tc_pair: tensor map encode failed (%d)", (int)r);
      P.drop0 = d0;
      P.n_ud = nd;
      P.n_uc = ncu;
      P.c0 = c0;
      const int64_t items = (int64_t)nd * P.n_pairs * ncu;
      const int grid = (int)(items < sms ? items : sms);
      {
        KTimer tm(s, "gram_stream_tc_pair_f16");
        gram_stream_tc_pair_kernel<<<grid, 256, smem, s>>>(map, P);
        tm.stop(s);
        count_launch();
      }
      rc = check_launch("gram_stream_tc_pair_kernel");
      if (rc) return rc;
    }
  }
  return XLMIMO_OK;
}

// K > 64 fused fp32: partials [drop][chunk][K(K+1)/2][2] into ws (fused_tc_pair_chunks(N) per drop).
int launch_fused_tc_pair(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                         cudaStream_t s) {
  FusedPairParams P;
  P.pos = pos;
  P.ws = ws;
  P.K = K;
  P.kind = a.kind;
  P.nb = (K + kPUsers - 1) / kPUsers;
  P.n_pairs = P.nb * (P.nb + 1) / 2;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = N;
  P.lambda = a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  P.n_chunks = fused_tc_pair_chunks(N);
  P.n_drops = n_drops;
  P.g = make_gen_const(a, N, kTaskE);
  const size_t smem = 1024 + (size_t)kPSlots * kPSlotBytes + (2 * kPSlots + 4) * 8 + 16 + 64 +
                      (size_t)kPGroups * 2 * kPUsers * 32;
  cudaFuncSetAttribute(gram_fused_tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = n_drops * P.n_pairs * P.n_chunks;
  const int grid = (int)(items < sms ? items : sms);
  gram_fused_tc_pair_kernel<<<grid, kPairThreads, smem, s>>>(P);
  return check_launch("gram_fused_tc_pair_kernel");
}

int launch_stream_tc(const float *H, int K, int64_t N, int64_t drop0, int nb, double *ws, cudaStream_t s) {
  auto enc = encode_fn();
  if (!enc) return set_error(XLMIMO_ECUDA, "stream_tc: cuTensorMapEncodeTiled unavailable");
  if (N % 128) return set_error(XLMIMO_EINVAL, "stream_tc: padded N must be a multiple of 128");
  CUtensorMap map;
  const cuuint64_t gdim[3] = {(cuuint64_t)kBoxK, (cuuint64_t)(2 * K), (cuuint64_t)(N / kBoxK) * nb};
  const cuuint64_t gstride[2] = {(cuuint64_t)kBoxK * 4, (cuuint64_t)kBoxK * 4 * 2 * K};
  const cuuint32_t box[3] = {(cuuint32_t)kBoxK, (cuuint32_t)(2 * K), 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)H, gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(XLMIMO_ECUDA, "stream_tc: tensor map encode failed (%d)", (int)r);
  StreamParams P;
  P.ws = ws;
  P.K = K;
  P.rb = rows_per_block(K);
  P.nblk = kRows / P.rb;
  P.n_mma = P.nblk > 1 ? kRows : (2 * K + 15) / 16 * 16;
  P.N = N;
  P.n_chunks = stream_tc_chunks(N);
  P.drop0 = drop0;
  P.nb = nb;
  uint32_t cols = 32;
  while (cols < (uint32_t)(3 * P.n_mma)) cols <<= 1;  // two accumulators + the running sum
  P.tmem_cols = cols;
  const size_t smem = 1024 + (size_t)kStages * kStageBytes + (2 * kStages + 4) * 8 + 16;
  cudaFuncSetAttribute(gram_stream_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = (int64_t)nb * P.n_chunks;
  const int grid = (int)(items < sms ? items : sms);
  gram_stream_tc_kernel<<<grid, kThreads, smem, s>>>(map, P);
  return check_launch("gram_stream_tc_kernel");
}

}  // namespace xlh
