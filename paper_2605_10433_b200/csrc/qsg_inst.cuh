// Explicit instantiation of decode_kernel<W, T, bp4, additive> for one W;
// included by qsg_inst_w*.cu with QSG_W defined (one W per translation unit
// so the build compiles them in parallel).
#include "qsg_internal.h"

#define QSG_FN2(w) kernel_ptr_w##w
#define QSG_FN(w) QSG_FN2(w)

namespace qsg {

template <int T, int NP>
static void *pick(bool bp4, bool add)
{
    if (bp4) return add ? (void *)decode_kernel<QSG_W, T, true, true, NP> : (void *)decode_kernel<QSG_W, T, true, false, NP>;
    return add ? (void *)decode_kernel<QSG_W, T, false, true, NP> : (void *)decode_kernel<QSG_W, T, false, false, NP>;
}

// np: compile-time qubit stride for the bicycle one-warp kernels at n_pad =
// 256 (every l in (64, 128], the BASELINE codes); 0 = run-time stride.
void *QSG_FN(QSG_W)(int T, bool bp4, bool add, int np)
{
#if QSG_W > 0
    if (T == 32 && np == 256) return pick<32, 256>(bp4, add);
    if (T == 32 && np == 128) return pick<32, 128>(bp4, add);
    if (T == 128 && np == 512) return pick<128, 512>(bp4, add);
    if (T == 128 && np == 1024) return pick<128, 1024>(bp4, add);
#endif
    if (T == 32) return pick<32, 0>(bp4, add);
    if (T == 128) return pick<128, 0>(bp4, add);
    return nullptr;
}

}  // namespace qsg
