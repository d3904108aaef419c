// Explicit instantiation of decode_kernel<W, T, bp4, additive> for one W;
// included by qsg_inst_w*.cu with QSG_W defined (one W per translation unit
// so the build compiles them in parallel).
#include "qsg_internal.h"

#define QSG_FN2(w) kernel_ptr_w##w
#define QSG_FN(w) QSG_FN2(w)

namespace qsg {

template <int T>
static void *pick(bool bp4, bool add)
{
    if (bp4) return add ? (void *)decode_kernel<QSG_W, T, true, true> : (void *)decode_kernel<QSG_W, T, true, false>;
    return add ? (void *)decode_kernel<QSG_W, T, false, true> : (void *)decode_kernel<QSG_W, T, false, false>;
}

void *QSG_FN(QSG_W)(int T, bool bp4, bool add)
{
    if (T == 32) return pick<32>(bp4, add);
    if (T == 128) return pick<128>(bp4, add);
    return nullptr;
}

}  // namespace qsg
