// kernels_inst.cu — instantiates the tile variants of ONE (body, dtype) pair.
//
// Compiled once per pair by build.py with
//   -DAMLT_BODY=<Gemm|Discount|Boost|Sqdiff|Eqcount|Thrcount>
//   -DAMLT_BODY_ID=<amlt_body> -DAMLT_T=<double|float|int> -DAMLT_DT=<amlt_dtype>
// so the (slow) template instantiations compile in parallel.
#include "variants.h"

#define AMLT_CAT2(a, b) a##b
#define AMLT_CAT(a, b) AMLT_CAT2(a, b)
#define AMLT_CAT4(a, b, c, d) AMLT_CAT(AMLT_CAT(a, b), AMLT_CAT(c, d))

namespace amltk {

void AMLT_CAT4(register_, AMLT_BODY, _, AMLT_DT)(Registry& reg) {
    using T = AMLT_T;
    using Body = AMLT_CAT(Body, AMLT_BODY)<T>;
    constexpr int ID = AMLT_BODY_ID;
    constexpr int DT = AMLT_DT;
    //                    TM TN WR WC BK ST  LOAD       MINB
    if constexpr (sizeof(T) == 8) {
        add_variant<Body, T, 8, 4, 8, 1, 16, 3, LOAD_TMA, 1>(reg, ID, DT, "t8x4_w8x1");
        add_variant<Body, T, 8, 2, 8, 1, 16, 3, LOAD_TMA, 2>(reg, ID, DT, "t8x2_w8x1");
        add_variant<Body, T, 4, 4, 8, 1, 16, 3, LOAD_TMA, 2>(reg, ID, DT, "t4x4_w8x1");
        add_variant<Body, T, 4, 4, 4, 1, 16, 4, LOAD_TMA, 3>(reg, ID, DT, "t4x4_w4x1");
        add_variant<Body, T, 4, 2, 4, 1, 16, 4, LOAD_TMA, 4>(reg, ID, DT, "t4x2_w4x1");
        add_variant<Body, T, 4, 4, 8, 1, 16, 3, LOAD_ELEM, 2>(reg, ID, DT, "t4x4_w8x1_u");
    } else {
        add_variant<Body, T, 8, 8, 4, 1, 32, 3, LOAD_TMA, 1>(reg, ID, DT, "t8x8_w4x1");
        add_variant<Body, T, 8, 4, 8, 1, 32, 3, LOAD_TMA, 1>(reg, ID, DT, "t8x4_w8x1");
        add_variant<Body, T, 4, 4, 8, 1, 32, 3, LOAD_TMA, 2>(reg, ID, DT, "t4x4_w8x1");
        add_variant<Body, T, 4, 4, 4, 1, 32, 4, LOAD_TMA, 3>(reg, ID, DT, "t4x4_w4x1");
        add_variant<Body, T, 4, 4, 8, 1, 32, 3, LOAD_ELEM, 2>(reg, ID, DT, "t4x4_w8x1_u");
    }
    // Thresholds indexed by i or by (i, j) (presets -ti / -tij): per-output
    // threshold state, smaller micro-tiles for the extra registers.
    if constexpr (UsesThreshold<Body>::value) {
        constexpr int TT = LOAD_TMA | LOAD_TOUT, TE = LOAD_ELEM | LOAD_TOUT;
        if constexpr (sizeof(T) == 8) {
            add_variant<Body, T, 4, 4, 8, 1, 16, 3, TT, 1>(reg, ID, DT, "t4x4_w8x1_ti");
            add_variant<Body, T, 4, 2, 4, 1, 16, 4, TT, 4>(reg, ID, DT, "t4x2_w4x1_ti");
            add_variant<Body, T, 4, 4, 8, 1, 16, 3, TE, 1>(reg, ID, DT, "t4x4_w8x1_ti_u");
        } else {
            add_variant<Body, T, 4, 4, 8, 1, 32, 3, TT, 2>(reg, ID, DT, "t4x4_w8x1_ti");
            add_variant<Body, T, 4, 4, 4, 1, 32, 4, TT, 3>(reg, ID, DT, "t4x4_w4x1_ti");
            add_variant<Body, T, 4, 4, 8, 1, 32, 3, TE, 2>(reg, ID, DT, "t4x4_w8x1_ti_u");
        }
    }
    BodyAux a;
    a.body = ID;
    a.dtype = DT;
    a.assign = &launch_assign<Body, T>;
    a.reduce = &launch_reduce<T>;
    a.assign_func = reinterpret_cast<const void*>(&mmlt_assign_kernel<Body, T>);
    a.reduce_func = reinterpret_cast<const void*>(&mmlt_splitk_reduce<T>);
    a.pack = &launch_pack<T>;
    a.pack_func = reinterpret_cast<const void*>(&mmlt_pack_kernel<T>);
    reg.aux.push_back(a);
}

}  // namespace amltk
