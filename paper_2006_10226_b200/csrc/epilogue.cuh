// epilogue.cuh — device helpers shared by the tcgen05 kernels (gemm_sm100.cu,
// depthwise_tc.cu): named barriers, TMEM loads, saturating packs, TMA stores and the
// fused fixed-point requantize of Eq. 5 over one 32-column chunk.
#pragma once

#include "common.cuh"

namespace qnn {

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int named_bar_and(int id, int n, int pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 q, %3, 0;\n\t"
      "bar.red.and.pred p, %1, %2, q;\n\t"
      "selp.s32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(id), "r"(n), "r"(pred)
      : "memory");
  return r;
}
// TMEM -> registers: 32 lanes x 32 columns, waited in the same asm so no use of
// the registers can be scheduled before the load completes.
__device__ __forceinline__ void tmem_load32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// Split TMEM load / wait for software pipelining: the wait takes the destination
// registers as in/out operands so no use of them can be scheduled before it.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}
__device__ __forceinline__ uint32_t pack4_u8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\t"
      "cvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\t"
      "cvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o)
      : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
__device__ __forceinline__ uint32_t pack4_s8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\t"
      "cvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\t"
      "cvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o)
      : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
__device__ __forceinline__ void tma_store_2d(const void* desc, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_dyn(int n) {   // n in {0, 1}
  if (n) bulk_wait_read<1>();
  else bulk_wait_read<0>();
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Fixed-point requantize of one accumulator column value (reading R1/R2/R15).
//   Fast UPWARD:    r = (mulhi(v, M) + c) >> t            c = 2^(t-1) + zp_out*2^t
//   Fast TONEAREST: r = sign(v) * ((mulhi(|v|, M) + c) >> t) + zp_out,  c = 2^(t-1)
//   Generic:        64-bit rounding shift by rsh (t holds -rsh, or t = rsh - 32)
template <int MODE, bool FAST>
__device__ __forceinline__ int32_t rq1(int32_t v, int32_t M, int32_t t, int32_t c, int32_t zp_out) {
  if (FAST) {
    if (MODE == 0) {
      return (__mulhi(v, M) + c) >> t;
    } else {
      const uint32_t a = v < 0 ? 0u - (uint32_t)v : (uint32_t)v;
      const int32_t m = (int32_t)((__umulhi(a, (uint32_t)M) + (uint32_t)c) >> t);
      return (v < 0 ? -m : m) + zp_out;
    }
  } else {
    const int rsh = t > 0 ? t + 32 : -t;
    return (int32_t)(rq_round((int64_t)v * M, rsh, MODE) + zp_out);
  }
}

// One 32-column chunk of one row: offsets, requantize, clamp; packed to 8-bit words
// (MODE 0/1) or kept as int32 (MODE 2, raw).  Parameters are read four columns per
// broadcast LDS.128: mt = {M, t} pairs, cc = c, off = folded offsets.
// Fused residual add (reading R19): R((res - zp_res) * s_res / s_out) with
// the residual's per-tensor fixed-point multiplier, added to the requantized conv value before
// the output clamp.  |res - zp_res| <= 255, so the 64-bit product never overflows.
struct ResTerm {
  int32_t M, rsh, zp, mode, s8;
};
__device__ __forceinline__ int32_t res_val(const ResTerm& t, uint32_t word, int byte) {
  const uint32_t b = (word >> (8 * byte)) & 0xFFu;
  const int32_t x = (t.s8 ? (int32_t)(int8_t)b : (int32_t)b) - t.zp;
  return (int32_t)rq_round((int64_t)x * t.M, t.rsh, t.mode);
}

template <int MODE, bool CLAMP, bool FAST, bool S8OUT, bool RES = false>
__device__ __forceinline__ void epi_chunk(const uint32_t (&v)[32], const int4* __restrict__ off4,
                                          const int4* __restrict__ mt4, const int4* __restrict__ c4,
                                          int32_t rterm, int32_t zp_out, int32_t lo, int32_t hi,
                                          uint32_t (&w)[8], int32_t* y, const uint32_t* rw = nullptr,
                                          const ResTerm* rt = nullptr) {
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    const int4 o = off4[q4];
    const int32_t offs[4] = {o.x, o.y, o.z, o.w};
    int32_t yy[4];
    if (MODE == 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) yy[u] = (int32_t)(v[q4 * 4 + u] + (uint32_t)offs[u] - (uint32_t)rterm);
    } else {
      const int4 mtA = mt4[q4 * 2], mtB = mt4[q4 * 2 + 1], cq = c4[q4];
      const int32_t Ms[4] = {mtA.x, mtA.z, mtB.x, mtB.z}, Ts[4] = {mtA.y, mtA.w, mtB.y, mtB.w};
      const int32_t Cs[4] = {cq.x, cq.y, cq.z, cq.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t vv = (int32_t)(v[q4 * 4 + u] + (uint32_t)offs[u] - (uint32_t)rterm);  // wrap-exact (R10)
        int32_t r = rq1<MODE, FAST>(vv, Ms[u], Ts[u], Cs[u], zp_out);
        if (RES) r += res_val(*rt, rw[q4], u);
        if (CLAMP) r = min(max(r, lo), hi);
        yy[u] = r;
      }
    }
    if (MODE == 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) y[q4 * 4 + u] = yy[u];
    } else {
      w[q4] = S8OUT ? pack4_s8(yy[0], yy[1], yy[2], yy[3]) : pack4_u8(yy[0], yy[1], yy[2], yy[3]);
    }
  }
}

// UPWARD fast path for one 32-column chunk of one row (see the header): two
// columns per LDS.128 of {M, t} pairs and per LDS.128 of K values.
template <bool CLAMP, bool S8OUT, bool RT, bool RES = false>
__device__ __forceinline__ void epi_chunk_up(const uint32_t (&v)[32], const int4* __restrict__ mt4,
                                             const longlong2* __restrict__ k2, int32_t rterm, int32_t lo,
                                             int32_t hi, uint32_t (&w)[8], const uint32_t* rw = nullptr,
                                             const ResTerm* rt = nullptr) {
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    int32_t yy[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int4 mt = mt4[q4 * 2 + h];
      const longlong2 kk = k2[q4 * 2 + h];
      int32_t v0 = (int32_t)v[q4 * 4 + 2 * h], v1 = (int32_t)v[q4 * 4 + 2 * h + 1];
      if (RT) {  // exact: sum_c A*(W - zp_W) is bounded by R10
        v0 -= rterm;
        v1 -= rterm;
      }
      int32_t r0 = mad_hi64(v0, mt.x, kk.x) >> mt.y;   // one IMAD.HI with the 64-bit K as addend
      int32_t r1 = mad_hi64(v1, mt.z, kk.y) >> mt.w;
      if (RES) {
        r0 += res_val(*rt, rw[q4], 2 * h);
        r1 += res_val(*rt, rw[q4], 2 * h + 1);
      }
      if (CLAMP) {
        r0 = min(max(r0, lo), hi);
        r1 = min(max(r1, lo), hi);
      }
      yy[2 * h] = r0;
      yy[2 * h + 1] = r1;
    }
    w[q4] = S8OUT ? pack4_s8(yy[0], yy[1], yy[2], yy[3]) : pack4_u8(yy[0], yy[1], yy[2], yy[3]);
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(pred));
  return pred != 0;
}


}  // namespace qnn
