// mttkrp_n5.cu — instantiations of mttkrp_sym_kernel for order 5 (split per
// order so the instantiations compile in parallel).
#include "mttkrp_kernel.cuh"

namespace systec {

template <int LPE, int VPL, int VW>
static KernelFn pos1_of(bool pos1, bool pf) {
    if (pf) return pos1 ? mttkrp_sym_kernel<5, LPE, VPL, VW, true, true> : mttkrp_sym_kernel<5, LPE, VPL, VW, false, true>;
    return pos1 ? mttkrp_sym_kernel<5, LPE, VPL, VW, true, false> : mttkrp_sym_kernel<5, LPE, VPL, VW, false, false>;
}

template <>
KernelFn pick_kernel<5>(int vw, int lpe, int vpl, bool pos1, bool pf) {
    if (vw == 1) {
        if (vpl != 1) return nullptr;
        switch (lpe) {
            case 1: return pos1_of<1, 1, 1>(pos1, pf);
            case 2: return pos1_of<2, 1, 1>(pos1, pf);
            case 4: return pos1_of<4, 1, 1>(pos1, pf);
            case 8: return pos1_of<8, 1, 1>(pos1, pf);
            case 16: return pos1_of<16, 1, 1>(pos1, pf);
            case 32: return pos1_of<32, 1, 1>(pos1, pf);
            default: return nullptr;
        }
    }
    switch (lpe * 8 + vpl) {  // (lanes per entry, float4 per lane)
        case 1 * 8 + 1: return pos1_of<1, 1, 4>(pos1, pf);
        case 1 * 8 + 2: return pos1_of<1, 2, 4>(pos1, pf);
        case 1 * 8 + 4: return pos1_of<1, 4, 4>(pos1, pf);
        case 2 * 8 + 1: return pos1_of<2, 1, 4>(pos1, pf);
        case 2 * 8 + 2: return pos1_of<2, 2, 4>(pos1, pf);
        case 2 * 8 + 4: return pos1_of<2, 4, 4>(pos1, pf);
        case 4 * 8 + 1: return pos1_of<4, 1, 4>(pos1, pf);
        case 4 * 8 + 2: return pos1_of<4, 2, 4>(pos1, pf);
        case 4 * 8 + 4: return pos1_of<4, 4, 4>(pos1, pf);
        case 8 * 8 + 1: return pos1_of<8, 1, 4>(pos1, pf);
        case 8 * 8 + 2: return pos1_of<8, 2, 4>(pos1, pf);
        case 8 * 8 + 4: return pos1_of<8, 4, 4>(pos1, pf);
        case 16 * 8 + 1: return pos1_of<16, 1, 4>(pos1, pf);
        case 16 * 8 + 2: return pos1_of<16, 2, 4>(pos1, pf);
        case 32 * 8 + 1: return pos1_of<32, 1, 4>(pos1, pf);
        default: return nullptr;
    }
}

template <int LPE, int VW>
static KernelFn naive_of(bool pf) {
    return pf ? mttkrp_sym_kernel<5, LPE, 1, VW, false, true, true> : mttkrp_sym_kernel<5, LPE, 1, VW, false, false, true>;
}

template <>
KernelFn pick_naive_kernel<5>(int vw, int lpe, bool pf) {
    if (vw == 4) {
        switch (lpe) {
            case 1: return naive_of<1, 4>(pf);
            case 2: return naive_of<2, 4>(pf);
            case 4: return naive_of<4, 4>(pf);
            case 8: return naive_of<8, 4>(pf);
            case 16: return naive_of<16, 4>(pf);
            case 32: return naive_of<32, 4>(pf);
            default: return nullptr;
        }
    }
    switch (lpe) {
        case 1: return naive_of<1, 1>(pf);
        case 2: return naive_of<2, 1>(pf);
        case 4: return naive_of<4, 1>(pf);
        case 8: return naive_of<8, 1>(pf);
        case 16: return naive_of<16, 1>(pf);
        case 32: return naive_of<32, 1>(pf);
        default: return nullptr;
    }
}

KernelFn ablation5(int abl) {
    switch (abl) {
        case 1: return mttkrp_sym_kernel<5, 4, 1, 4, true, false, false, 1>;
        case 2: return mttkrp_sym_kernel<5, 4, 1, 4, true, false, false, 2>;
        case 3: return mttkrp_sym_kernel<5, 4, 1, 4, true, false, false, 3>;
        default: return nullptr;
    }
}

KernelFn occupancy5(bool pos1) {
    return pos1 ? mttkrp_sym_kernel_occ<5, 4, 1, 4, true, 4> : mttkrp_sym_kernel_occ<5, 4, 1, 4, false, 4>;
}

template <>
KernelFn pick_full_kernel<5>(int lpe, bool pos1, bool occ) {
    if (occ) {
        if (lpe != 4) return nullptr;
        return pos1 ? mttkrp_sym_kernel_occ<5, 4, 1, 4, true, 4, 16> : mttkrp_sym_kernel_occ<5, 4, 1, 4, false, 4, 16>;
    }
    switch (lpe) {
        case 4: return pos1 ? mttkrp_sym_kernel<5, 4, 1, 4, true, false, false, 0, 16> : mttkrp_sym_kernel<5, 4, 1, 4, false, false, false, 0, 16>;
        case 8: return pos1 ? mttkrp_sym_kernel<5, 8, 1, 4, true, false, false, 0, 32> : mttkrp_sym_kernel<5, 8, 1, 4, false, false, false, 0, 32>;
        default: return nullptr;
    }
}

template <>
KernelFn pick_full_v8_kernel<5>(bool pos1) {
    return pos1 ? mttkrp_sym_kernel<5, 2, 1, 8, true, false, false, 0, 16>
                : mttkrp_sym_kernel<5, 2, 1, 8, false, false, false, 0, 16>;
}

template <>
KernelFn pick_full_naive_kernel<5>(int lpe) {
    switch (lpe) {
        case 4: return mttkrp_sym_kernel<5, 4, 1, 4, false, false, true, 0, 16>;
        case 8: return mttkrp_sym_kernel<5, 8, 1, 4, false, false, true, 0, 32>;
        default: return nullptr;
    }
}

}  // namespace systec
