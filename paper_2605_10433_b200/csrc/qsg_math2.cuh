// Paired (f32x2) evaluation of the fp32 recipes in qsg_math.cuh.
//
// sm_100 issues FFMA2 / FADD2 / FMUL2: one warp instruction performs two
// independent IEEE binary32 fused multiply-adds / adds / multiplies, each
// rounded exactly like its scalar counterpart.  The kernels spend most of
// their issue slots on these recipes, and they always evaluate them on
// independent pairs (the two factors F(S_Z), F(S_X) of a qubit; the
// exponentials, prefix / suffix steps and logarithms of a BP4 check), so
// every function below is the scalar recipe
// applied to both halves of an F2, operation for operation: the results are
// bit-identical to two calls of the scalar version (and therefore to the
// oracle).  Integer / bit manipulations and selects run per half; there is
// no packed min/max.
#pragma once

#include <stdint.h>

#include "qsg_math.cuh"

namespace qsg {

struct F2 {
    unsigned long long v;
};

__device__ __forceinline__ F2 pk(float a, float b)
{
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ F2 bc(float c) { return pk(c, c); }
__device__ __forceinline__ float lo(F2 r)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r.v));
    return a;
}
__device__ __forceinline__ float hi(F2 r)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r.v));
    return b;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c)
{
    F2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return d;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b)
{
    F2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b)
{
    F2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
// a * b.  ptxas contracts an f32x2 multiply with a following f32x2 add into
// one FFMA2 even for .rn-qualified PTX (and with -fmad=false), which would
// change the rounding; the recipes are therefore written so that every
// product feeding an addition is either exact (scaling by 2^k) or an
// explicit fma in the scalar recipe too.
__device__ __forceinline__ F2 mul2(F2 a, F2 b)
{
    F2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}

// exp_neg on both halves (qsg_math.cuh exp_neg).
__device__ __forceinline__ F2 exp_neg2(F2 x)
{
    const F2 t = fma2(x, bc(kLog2e), bc(kMagic));
    const F2 k = sub2(t, bc(kMagic));
    F2 r = fma2(k, bc(-kLn2Hi), x);
    r = fma2(k, bc(-kLn2Lo), r);
    F2 p = fma2(bc(0.0013751407f), r, bc(0.008368917f));
    p = fma2(p, r, bc(0.041669533f));
    p = fma2(p, r, bc(0.16666518f));
    p = fma2(p, r, bc(0.49999988f));
    p = fma2(p, r, bc(1.0f));
    p = fma2(p, r, bc(1.0f));
    const F2 s = pk(u2f((f2u(lo(t)) + (127u - kMagicBits)) << 23), u2f((f2u(hi(t)) + (127u - kMagicBits)) << 23));
    return mul2(p, s);
}

// log1p_01 on both halves.
__device__ __forceinline__ F2 log1p_01_poly2(F2 t)
{
    F2 p = fma2(bc(-0.003227271f), t, bc(0.019791102f));
    p = fma2(p, t, bc(-0.05688295f));
    p = fma2(p, t, bc(0.106008776f));
    p = fma2(p, t, bc(-0.15308061f));
    p = fma2(p, t, bc(0.19678909f));
    p = fma2(p, t, bc(-0.24955378f));
    p = fma2(p, t, bc(0.33330205f));
    p = fma2(p, t, bc(-0.49999923f));
    return fma2(p, t, bc(1.0f));
}
__device__ __forceinline__ F2 log1p_01_2(F2 t) { return mul2(t, log1p_01_poly2(t)); }
// -P(t): every coefficient negated.  Rounding to nearest is symmetric in the
// sign, so each step is exactly the negative of log1p_01_poly2's, and
// fma(t, -P, L) == fma(-t, P, L) bit for bit -- without the negation op.
__device__ __forceinline__ F2 log1p_01_npoly2(F2 t)
{
    F2 p = fma2(bc(0.003227271f), t, bc(-0.019791102f));
    p = fma2(p, t, bc(0.05688295f));
    p = fma2(p, t, bc(-0.106008776f));
    p = fma2(p, t, bc(0.15308061f));
    p = fma2(p, t, bc(-0.19678909f));
    p = fma2(p, t, bc(0.24955378f));
    p = fma2(p, t, bc(-0.33330205f));
    p = fma2(p, t, bc(0.49999923f));
    return fma2(p, t, bc(-1.0f));
}
// y >= 0 ? a : b as FSETP + FSEL (the compiler otherwise builds the selected
// pair with predicated moves, three to four per pair).
__device__ __forceinline__ float sel_ge0(float y, float a, float b)
{
    float d;
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, 0f00000000;\n\tselp.f32 %0, %2, %3, p;\n\t}"
        : "=f"(d) : "f"(y), "f"(a), "f"(b));
    return d;
}

// (a & 0x7fffff) | 0x3f800000 as ONE LOP3: with both masks as immediates
// ptxas splits it in two; the OR constant is kept in a register instead.
__device__ __forceinline__ uint32_t mant_one(uint32_t a)
{
    uint32_t k, d;
    asm volatile("mov.b32 %0, 0x3f800000;" : "=r"(k));
    asm("lop3.b32 %0, %1, 0x007fffff, %2, 0xea;" : "=r"(d) : "r"(a), "r"(k));
    return d;
}

// e ln2 + log1p(m - 1) for u = 2^e m on both halves (log_pos).
__device__ __forceinline__ F2 log_pos2(F2 u)
{
    const uint32_t a = f2u(lo(u)), b = f2u(hi(u));
    const F2 fe = sub2(pk(u2f(kMagicBits + ((a >> 23) - 127u)), u2f(kMagicBits + ((b >> 23) - 127u))), bc(kMagic));
    const F2 f = sub2(pk(u2f(mant_one(a)), u2f(mant_one(b))), bc(1.0f));
    return fma2(fe, bc(kLn2Hi), fma2(fe, bc(kLn2Lo), log1p_01_2(f)));
}

// vn_F(y0, kapc), vn_F(y1, kapc).
__device__ __forceinline__ F2 vn_F2(float y0, float y1, F2 kapc2)
{
    const F2 x = pk(-fminf(fabsf(y0), 87.0f), -fminf(fabsf(y1), 87.0f));
    const F2 q = exp_neg2(x);
    const F2 af = fma2(kapc2, q, bc(1.0f)), aa = add2(kapc2, q);
    const F2 A = pk(sel_ge0(y0, lo(af), lo(aa)), sel_ge0(y1, hi(af), hi(aa)));
    return fma2(q, log1p_01_npoly2(q), log_pos2(A));  // log(A) - q P(q), one rounding
}

// rcp_rn on both halves: two MUFU.RCP seeds, the Newton step on FFMA2.
__device__ __forceinline__ F2 rcp_rn2(F2 o)
{
    float y0, y1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(lo(o)));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(hi(o)));
    const F2 y = pk(y0, y1);
    return fma2(y, fma2(sub2(bc(0.0f), o), y, bc(1.0f)), y);  // 0 - o = -o exactly
}

// BP4 magnitudes of two edges from their (E, O) pairs.
__device__ __forceinline__ F2 bp4_out2(F2 EOa, F2 EOb)
{
    const F2 y = rcp_rn2(pk(fmaxf(hi(EOa), 1e-30f), fmaxf(hi(EOb), 1e-30f)));
    const F2 L = log_pos2(mul2(pk(lo(EOa), lo(EOb)), y));
    return pk(fminf(fmaxf(lo(L), kPhi50), kPhiTiny), fminf(fmaxf(hi(L), kPhi50), kPhiTiny));
}

// BP4 product-form magnitudes (qsg_math.cuh bp4_mags) for a check of
// compile-time degree D (even), laid out so that every FFMA2 operand is a
// register pair as produced, its swapped halves or one broadcast register
// (all free operand forms on sm_100; packing two values from different pairs
// costs a move, which lands on the FMA pipe this kernel is bound by):
//   prefix pair PA_j = (A_j, B_j):  PA_{j+1} = fma(s_j, swap(PA_j), PA_j)
//   suffix pair SC_e = (C_e, D_e):  SC_{e-1} = fma(s_e, swap(SC_e), SC_e)
//   merge  (E_e, O_e) = fma(A_e, SC_e, B_e * swap(SC_e))
// (halves: A + s B, B + s A / C + s D, D + s C / A C + B D, A D + B C -- the
// scalar recipe's operations, bit-identical).  Exponentials run on edge
// pairs, the ratio E * rcp(O) as two scalar products, and the reciprocal and
// logarithm of two edges as pairs.  Edges are finished as soon as their
// prefix and suffix exist (two per step from the middle), which keeps few
// partial products live.
__device__ __forceinline__ F2 swp(F2 a) { return pk(hi(a), lo(a)); }

__device__ __forceinline__ F2 bp4_merge(F2 PA, F2 SC)
{
    return fma2(bc(lo(PA)), SC, mul2(bc(hi(PA)), swp(SC)));  // (E, O)
}

// magnitudes of two edges from their (E, O) pairs
__device__ __forceinline__ F2 bp4_out2s(F2 EOa, F2 EOb)
{
    const F2 y = rcp_rn2(pk(fmaxf(hi(EOa), 1e-30f), fmaxf(hi(EOb), 1e-30f)));
    const F2 L = log_pos2(pk(lo(EOa) * lo(y), lo(EOb) * hi(y)));
    return pk(fminf(fmaxf(lo(L), kPhi50), kPhiTiny), fminf(fmaxf(hi(L), kPhi50), kPhiTiny));
}

template <int D>
__device__ __forceinline__ void bp4_mags_fixed(const float (&x)[D], float (&mag)[D])
{
    static_assert(D % 2 == 0, "paired exponentials need an even degree");
    float s[D];
#pragma unroll
    for (int k = 0; k < D; k += 2) {
        const F2 e = exp_neg2(pk(-x[k], -x[k + 1]));
        s[k] = lo(e); s[k + 1] = hi(e);
    }
    F2 PA[D], SC[D];
    PA[0] = pk(1.0f, 0.0f);
    SC[D - 1] = pk(1.0f, 0.0f);
#pragma unroll
    for (int j = 0; j + 1 < D; ++j) {
        PA[j + 1] = fma2(bc(s[j]), swp(PA[j]), PA[j]);
        SC[D - 2 - j] = fma2(bc(s[D - 1 - j]), swp(SC[D - 1 - j]), SC[D - 1 - j]);
        if (D - 2 - j < j + 1) {  // new edges D - 2 - j and j + 1
            const int a = D - 2 - j, b = j + 1;
            const F2 m = bp4_out2s(bp4_merge(PA[a], SC[a]), bp4_merge(PA[b], SC[b]));
            mag[a] = lo(m);
            mag[b] = hi(m);
        }
    }
}

}  // namespace qsg
