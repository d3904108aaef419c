// Paired (f32x2) evaluation of the fp32 recipes in qsg_math.cuh.
//
// sm_100 issues FFMA2 / FADD2 / FMUL2: one warp instruction performs two
// independent IEEE binary32 fused multiply-adds / adds / multiplies, each
// rounded exactly like its scalar counterpart.  The kernels spend most of
// their issue slots on these recipes, and they always evaluate them on
// independent pairs (the two factors F(S_Z), F(S_X) of a qubit, the phi of
// edges k and k+1 of a check), so every function below is the scalar recipe
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

// e ln2 + log1p(m - 1) for u = 2^e m on both halves (log_pos; phi_lo's log).
__device__ __forceinline__ F2 log_pos2(F2 u)
{
    const uint32_t a = f2u(lo(u)), b = f2u(hi(u));
    const F2 fe = sub2(pk(u2f(kMagicBits + ((a >> 23) - 127u)), u2f(kMagicBits + ((b >> 23) - 127u))), bc(kMagic));
    const F2 f = sub2(pk(u2f((a & 0x007fffffu) | 0x3f800000u), u2f((b & 0x007fffffu) | 0x3f800000u)), bc(1.0f));
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

// phi_hi / phi_lo / phi on both halves (BP4).
__device__ __forceinline__ F2 phi_hi2(F2 x)
{
    const F2 t = exp_neg2(sub2(bc(0.0f), x));
    const F2 u = mul2(t, t);
    F2 S = fma2(bc(0.15731367f), u, bc(0.06506128f));
    S = fma2(S, u, bc(0.11467144f));
    S = fma2(S, u, bc(0.1426422f));
    S = fma2(S, u, bc(0.20000467f));
    S = fma2(S, u, bc(0.3333333f));
    const F2 tt = add2(t, t);
    return fma2(mul2(tt, u), S, tt);
}
__device__ __forceinline__ F2 phi_lo2(F2 x)
{
    const F2 lg = log_pos2(x);
    const F2 v = mul2(x, x);
    F2 H = fma2(bc(-2.4306313e-05f), v, bc(0.0003411371f));
    H = fma2(H, v, bc(-0.0048610563f));
    H = fma2(H, v, bc(0.083333336f));
    return fma2(v, H, sub2(bc(kLn2f), lg));
}
__device__ __forceinline__ F2 phi2(F2 x)
{
    const F2 a = phi_hi2(x), b = phi_lo2(x);
    return pk(lo(x) < kLn2f ? lo(b) : lo(a), hi(x) < kLn2f ? hi(b) : hi(a));
}

}  // namespace qsg
