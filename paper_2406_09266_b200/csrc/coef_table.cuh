// coef_table.cuh — the per-equality-pattern multiplicity coefficients of the
// symmetric MTTKRP, generated at compile time and placed in __constant__.
//
// Paper basis.  A stored canonical entry c_0 <= ... <= c_{n-1} (Def. Canonical,
// PAPER.md:162-167) belongs to exactly one equivalence group E:
// the partition of its positions into runs of equal indices.  We encode E as a
// pattern code with bit t set iff c_t == c_{t+1}.  Symmetrisation issues one
// assignment per member of the unique symmetry group S_P|E (PAPER.md:381-386,
// fig:symmetrization_pseudocode PAPER.md:402-420); for MTTKRP all members that
// put the same index value into the output position write the same product, so
// the distributive grouping of PAPER.md:577-591 merges them into one update with
// an integer factor.  The members that put run u's value first are the distinct
// permutations of the remaining multiset:
//     coef[u] = (n-1)! * m_u / prod_w m_w!      at the first position of run u,
//     coef[t] = 0                                at the other positions of a run.
// The factors are looked up, not branched on — the consolidated conditional
// block + simplicial lookup table of PAPER.md:506-553 (whose printed key is
// garbled, reading X2; we index by the bitmask instead).
#pragma once

namespace systec {

constexpr int kMaxOrder = 5;

struct CoefTable {
    float v[kMaxOrder - 1][1 << (kMaxOrder - 1)][kMaxOrder];  // [n-2][code][pos]
};

constexpr long long cfact(int k) { return k <= 1 ? 1 : k * cfact(k - 1); }

constexpr CoefTable make_coef_table() {
    CoefTable T{};
    for (int n = 2; n <= kMaxOrder; ++n) {
        for (int code = 0; code < (1 << (n - 1)); ++code) {
            // run id and run size of every position
            int run_of[kMaxOrder] = {};
            int run_size[kMaxOrder] = {};
            int nruns = 0;
            for (int t = 0; t < n; ++t) {
                const bool joins = t > 0 && ((code >> (t - 1)) & 1);
                if (!joins) ++nruns;
                run_of[t] = nruns - 1;
                run_size[nruns - 1] += 1;
            }
            long long denom = 1;
            for (int u = 0; u < nruns; ++u) denom *= cfact(run_size[u]);
            for (int t = 0; t < n; ++t) {
                const bool first = t == 0 || !((code >> (t - 1)) & 1);
                const long long num = cfact(n - 1) * run_size[run_of[t]];
                T.v[n - 2][code][t] = first ? static_cast<float>(num / denom) : 0.0f;
            }
        }
    }
    return T;
}

constexpr CoefTable kCoefHost = make_coef_table();

// compile-time spot checks against the hand-expanded Listing 6
static_assert(kCoefHost.v[1][0][0] == 2 && kCoefHost.v[1][0][1] == 2 && kCoefHost.v[1][0][2] == 2, "n=3 <<");
static_assert(kCoefHost.v[1][1][0] == 2 && kCoefHost.v[1][1][1] == 0 && kCoefHost.v[1][1][2] == 1, "n=3 =<");
static_assert(kCoefHost.v[1][2][0] == 1 && kCoefHost.v[1][2][1] == 2 && kCoefHost.v[1][2][2] == 0, "n=3 <=");
static_assert(kCoefHost.v[1][3][0] == 1 && kCoefHost.v[1][3][1] == 0 && kCoefHost.v[1][3][2] == 0, "n=3 ==");
static_assert(kCoefHost.v[3][0][4] == 24 && kCoefHost.v[3][15][0] == 1, "n=5 extremes");

}  // namespace systec
