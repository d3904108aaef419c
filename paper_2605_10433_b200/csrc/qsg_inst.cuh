// Explicit instantiation of decode_kernel<W, T, bp4, additive> for one W;
// included by qsg_inst_w*.cu with QSG_W defined (one W per translation unit
// so the build compiles them in parallel).
#include "qsg_internal.h"

#define QSG_FN2(w) kernel_ptr_w##w
#define QSG_FN(w) QSG_FN2(w)

namespace qsg {

template <int T, int NP>
static void *pick(bool bp4, bool add, bool lean = false)
{
#if QSG_W > 0
    // lean instances (qsg_kernel.cuh): marginal qubit update, compile-time stride
    if constexpr (NP > 0) {
        if (lean && !add)
            return bp4 ? (void *)decode_kernel<QSG_W, T, true, false, NP, true>
                       : (void *)decode_kernel<QSG_W, T, false, false, NP, true>;
    }
#endif
    if (bp4) return add ? (void *)decode_kernel<QSG_W, T, true, true, NP> : (void *)decode_kernel<QSG_W, T, true, false, NP>;
    return add ? (void *)decode_kernel<QSG_W, T, false, true, NP> : (void *)decode_kernel<QSG_W, T, false, false, NP>;
}

// np: bicycle kernels (W > 0): compile-time qubit stride n_pad (0 = run
// time; those and the generic kernels have no lean instance, `lean` is then
// ignored -- lean_kernel_exists in qsg_abi.cu mirrors this list); generic kernels (W == 0): the node-degree bound (8, 12, 16, 24 or
// 32) that sizes their register arrays.
void *QSG_FN(QSG_W)(int T, bool bp4, bool add, int np, bool lean)
{
#if QSG_W == 0
    if (T != 32 && T != 128) return nullptr;
    if (np <= 8) return T == 32 ? pick<32, 8>(bp4, add) : pick<128, 8>(bp4, add);
    if (np <= 12) return T == 32 ? pick<32, 12>(bp4, add) : pick<128, 12>(bp4, add);
    if (np <= 16) return T == 32 ? pick<32, 16>(bp4, add) : pick<128, 16>(bp4, add);
    if (np <= 24) return T == 32 ? pick<32, 24>(bp4, add) : pick<128, 24>(bp4, add);
    return T == 32 ? pick<32, 32>(bp4, add) : pick<128, 32>(bp4, add);
#else
    if (T == 32 && np == 256) return pick<32, 256>(bp4, add, lean);
    if (T == 32 && np == 128) return pick<32, 128>(bp4, add, lean);
    if (T == 128 && np == 512) return pick<128, 512>(bp4, add, lean);
    if (T == 64 && np == 512) return pick<64, 512>(bp4, add, lean);
    if (T == 64) return pick<64, 0>(bp4, add);
    if (T == 128 && np == 1024) return pick<128, 1024>(bp4, add, lean);
    if (T == 32) return pick<32, 0>(bp4, add);
    if (T == 128) return pick<128, 0>(bp4, add);
    return nullptr;
#endif
}

}  // namespace qsg
