// register_all.cu — collects the per-(body, dtype) registration functions
// compiled from kernels_inst.cu (dtype codes: 0 f64, 1 f32, 2 i32).
#include "variants.h"

namespace amltk {

#define AMLT_PAIRS(X)                                                                       \
    X(Gemm, 0) X(Discount, 0) X(Boost, 0) X(Sqdiff, 0) X(Eqcount, 0) X(Thrcount, 0)       \
    X(Gemm, 1) X(Discount, 1) X(Boost, 1) X(Sqdiff, 1) X(Eqcount, 1) X(Thrcount, 1)       \
    X(Eqcount, 2) X(Thrcount, 2)

#define AMLT_DECL(B, D) void register_##B##_##D(Registry&);
AMLT_PAIRS(AMLT_DECL)
void register_dmma_gemm(Registry&);
void register_tcgen05_gemm(Registry&);
void register_ozaki_gemm(Registry&);
void register_theta_discount(Registry&);
void register_swar_eqcount(Registry&);

void register_all(Registry& reg) {
#define AMLT_CALL(B, D) register_##B##_##D(reg);
    AMLT_PAIRS(AMLT_CALL)
    register_dmma_gemm(reg);
    register_tcgen05_gemm(reg);
    register_ozaki_gemm(reg);
    register_theta_discount(reg);
    register_swar_eqcount(reg);
}

}  // namespace amltk
