// Update rules in f64 with a cast on store, reproducing sgd.cpp:46-88
// operation by operation. Every product/sum is an explicit round-to-nearest
// intrinsic so nvcc cannot contract a*b+c into an FMA: the reference's x86-64
// build rounds each operation separately, and parity is bitwise.
#pragma once

#include "common.cuh"

namespace synk {

struct RuleParams {
    int rule;
    double lr;
    double h0, h1, h2;  // momentum: mu | rmsprop: rho, eps | adam: beta1, beta2, eps
    double c1, c2;      // adam bias corrections 1 - beta^t, computed on the host (std::pow)
};

// p, a0, a1 in/out (f64 views of the stored T values); g = gradient (stored T).
__device__ __forceinline__ void rule_update(const RuleParams& rp, double& p, double& a0,
                                            double& a1, double g) {
    switch (rp.rule) {
    case SYNK_RULE_SGD:  // sgd.cpp:49
        p = __dsub_rn(p, __dmul_rn(rp.lr, g));
        break;
    case SYNK_RULE_MOMENTUM: {  // sgd.cpp:56-59
        double vn = __dsub_rn(__dmul_rn(rp.h0, a0), __dmul_rn(rp.lr, g));
        a0 = vn;
        p = __dsub_rn(__dadd_rn(p, __dmul_rn(rp.h0, vn)), __dmul_rn(rp.lr, g));
        break;
    }
    case SYNK_RULE_RMSPROP: {  // sgd.cpp:66-70
        double an = __dadd_rn(__dmul_rn(rp.h0, a0), __dmul_rn(__dmul_rn(__dsub_rn(1.0, rp.h0), g), g));
        a0 = an;
        p = __dsub_rn(p, __ddiv_rn(__dmul_rn(rp.lr, g), __dsqrt_rn(__dadd_rn(an, rp.h1))));
        break;
    }
    default: {  // SYNK_RULE_ADAM, sgd.cpp:79-86
        double mn = __dadd_rn(__dmul_rn(rp.h0, a0), __dmul_rn(__dsub_rn(1.0, rp.h0), g));
        double vn = __dadd_rn(__dmul_rn(rp.h1, a1), __dmul_rn(__dmul_rn(__dsub_rn(1.0, rp.h1), g), g));
        a0 = mn;
        a1 = vn;
        double num = __dmul_rn(rp.lr, __ddiv_rn(mn, rp.c1));
        double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vn, rp.c2)), rp.h2);
        p = __dsub_rn(p, __ddiv_rn(num, den));
        break;
    }
    }
}

// The same with the rule fixed at compile time (RULE < 0: rp.rule at run
// time): the streaming update loop then carries one rule's code only.
template <int RULE>
__device__ __forceinline__ void rule_update_t(const RuleParams& rp, double& p, double& a0, double& a1, double g) {
    if constexpr (RULE < 0) {
        rule_update(rp, p, a0, a1, g);
    } else {
        RuleParams r = rp;
        r.rule = RULE;
        if constexpr (RULE == SYNK_RULE_SGD) {
            p = __dsub_rn(p, __dmul_rn(rp.lr, g));
        } else {
            rule_update(r, p, a0, a1, g);  // switch folds: r.rule is a constant
        }
    }
}

inline int rule_aux_count(int rule) {
    return rule == SYNK_RULE_SGD ? 0 : (rule == SYNK_RULE_ADAM ? 2 : 1);
}

}  // namespace synk
