// Test harness: the PRODUCT's fp32 recipes (qsg_math.cuh) compiled for the
// host, so tests/test_oracle_math.py can check they equal the oracle's
// independent copy bit-for-bit.
#include <math.h>
#include <stdint.h>
#include "../../paper_2605_10433_b200/csrc/qsg_math.cuh"

extern "C" void qsg_math_host_batch(int32_t which, const float *x, const float *y, float *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) {
        switch (which) {
        case 0: out[i] = qsg::exp_neg(x[i]); break;
        case 1: out[i] = qsg::log1p_01(x[i]); break;
        case 2: out[i] = qsg::log1p_pos(x[i]); break;
        case 3: out[i] = qsg::expm1_pos(x[i]); break;
        case 4: out[i] = qsg::logaddexp(x[i], y[i]); break;
        case 6: out[i] = qsg::vn_F(x[i], (float)exp(-(double)y[i])); break;  // kapc as the ABI computes it
        default: out[i] = 0.0f;
        }
    }
}

// One BP4 check: the product copy of the product-form magnitudes.
extern "C" void qsg_bp4_host(const float *x, int32_t d, float *out)
{
    if (d >= 1 && d <= qsg::kBp4MaxDeg) qsg::bp4_mags(x, d, out);
}
