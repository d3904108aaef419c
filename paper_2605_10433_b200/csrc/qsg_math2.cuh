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
    const F2 A = pk(y0 >= 0.0f ? lo(af) : lo(aa), y1 >= 0.0f ? hi(af) : hi(aa));
    return fma2(sub2(bc(0.0f), q), log1p_01_poly2(q), log_pos2(A));
}

// rcp3 on both halves (o > 0).
__device__ __forceinline__ F2 rcp3_2(F2 o)
{
    F2 y = pk(u2f(0x7ef311c3u - f2u(lo(o))), u2f(0x7ef311c3u - f2u(hi(o))));
    const F2 no = sub2(bc(0.0f), o);  // -o, exact
#pragma unroll
    for (int i = 0; i < 3; ++i) y = fma2(y, fma2(no, y, bc(1.0f)), y);
    return y;
}

// BP4 magnitudes of two edges from their (E, O) pairs.
__device__ __forceinline__ F2 bp4_out2(F2 EOa, F2 EOb)
{
    const F2 y = rcp3_2(pk(fmaxf(hi(EOa), 1e-30f), fmaxf(hi(EOb), 1e-30f)));
    const F2 L = log_pos2(mul2(pk(lo(EOa), lo(EOb)), y));
    return pk(fminf(fmaxf(lo(L), kPhi50), kPhiTiny), fminf(fmaxf(hi(L), kPhi50), kPhiTiny));
}

// BP4 product-form magnitudes (qsg_math.cuh bp4_mags) for a check of
// compile-time degree D (even): exponentials on edge pairs, the prefix and
// suffix recurrences side by side on FFMA2 (prefix in the low half, suffix
// in the high half), the per-edge merge as an FMUL2 + FFMA2 (E, O) pair, and
// the reciprocal, ratio and logarithm of two edges as pairs.  Each half performs exactly the scalar
// recipe's operations (bit-identical).
template <int D>
__device__ __forceinline__ void bp4_mags_fixed(const float (&x)[D], float (&mag)[D])
{
    static_assert(D % 2 == 0, "paired exponentials need an even degree");
    float s[D], A[D], B[D], C[D], Dd[D];
#pragma unroll
    for (int k = 0; k < D; k += 2) {
        const F2 e = exp_neg2(pk(-x[k], -x[k + 1]));
        s[k] = lo(e); s[k + 1] = hi(e);
    }
    A[0] = 1.0f; B[0] = 0.0f; C[D - 1] = 1.0f; Dd[D - 1] = 0.0f;
    F2 P = bc(1.0f), Q = bc(0.0f);  // (A_j, C_{D-1-j}), (B_j, D_{D-1-j})
    // edges are merged as soon as their prefix (step e - 1) and suffix
    // (step D - 2 - e) exist -- two per step from step D/2 - 1, which keeps
    // fewer partial products live -- and finished as a pair
    auto merge = [&](int e) {
        const F2 t = mul2(bc(B[e]), pk(Dd[e], C[e]));            // (B D, B C)
        return fma2(bc(A[e]), pk(C[e], Dd[e]), t);               // (E_e, O_e)
    };
#pragma unroll
    for (int j = 0; j + 1 < D; ++j) {
        const F2 S = pk(s[j], s[D - 1 - j]);
        const F2 Pn = fma2(S, Q, P), Qn = fma2(S, P, Q);
        P = Pn; Q = Qn;
        A[j + 1] = lo(P); B[j + 1] = lo(Q); C[D - 2 - j] = hi(P); Dd[D - 2 - j] = hi(Q);
        if (D - 2 - j < j + 1) {  // new edges D - 2 - j and j + 1
            const F2 m = bp4_out2(merge(D - 2 - j), merge(j + 1));
            mag[D - 2 - j] = lo(m);
            mag[j + 1] = hi(m);
        }
    }
}

}  // namespace qsg
