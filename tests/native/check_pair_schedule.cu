// Host-side check of the static row-owner pair schedule of kernel_tiled.cuh (PairSched<G,S>): for every tier the
// (lane, step) -> pair mapping must cover every off-diagonal pair (a, c), 1 <= c < a <= CAP-1, exactly once
// (column 0 is the padding row and must never be written).  Mirrors the case analysis of the kernel's pair phase.
#include <cstdio>
#include <vector>
#include "kernel_tiled.cuh"

template <int G, int S>
static int check()
{
    using PS = PairSched<G, S>;
    constexpr int CAP = G * S;
    std::vector<int> seen(CAP * CAP, 0);
    int bad = 0;
    for (int lg = 0; lg < G; ++lg) {
        int rowi[S];
        for (int s = 0; s < S; ++s)
            rowi[s] = s * G + ((s & 1) ? (G - 1 - lg) : lg);
        for (int k = 0; k < PS::NIT; ++k) {
            const int h = PS::h_of(k), t = PS::t_of(k), kind = PS::kind(k);
            const int s1 = (h < PS::NH) ? 2 * h + 1 : S - 1, s0 = (h < PS::NH) ? 2 * h : S - 1;
            const int c1 = t, c0 = (h < PS::NH) ? PS::T(h) - 1 - t : t;
            int a = -1, c = -1;
            if (kind == PS::ALL1) { a = rowi[s1]; c = c1; }
            else if (kind == PS::ALL0) { a = rowi[s0]; c = c0; }
            else if (kind == PS::MIXED) {
                const bool pr = lg < (2 * h + 2) * G - 1 - t;
                if (pr) { a = rowi[s1]; c = c1; }
                else if (c0 > 0) { a = rowi[s0]; c = c0; }
            } else if (t < rowi[S - 1]) { a = rowi[S - 1]; c = c1; }
            if (a < 0)
                continue; // idle lane at this step
            if (c < 1 || c >= a || a >= CAP) { ++bad; continue; }
            ++seen[a * CAP + c];
        }
    }
    for (int a = 1; a < CAP; ++a)
        for (int c = 1; c < a; ++c)
            if (seen[a * CAP + c] != 1)
                ++bad;
    std::printf("G=%d S=%d steps=%d pairs=%d %s\n", G, S, PS::NIT, (CAP - 1) * (CAP - 2) / 2, bad ? "FAIL" : "ok");
    return bad;
}

int main()
{
    int bad = 0;
    bad += check<4, 3>();
    bad += check<8, 3>();
    bad += check<16, 2>();
    bad += check<16, 3>();
    bad += check<32, 2>();
    bad += check<8, 4>();
    bad += check<4, 2>();
    bad += check<8, 5>();
    return bad ? 1 : 0;
}
