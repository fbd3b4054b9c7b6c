// Level-independent FMM translation operators in the real semi-normalised
// basis of harmonics.h (built once on the host in FP64, stored FP32 on the
// device).  Box-scaled coefficients make every operator independent of the
// tree level:
//   M2M: 8 child octants -> parent           mu_p  = T_oct  mu_c
//   L2L: parent -> 8 child octants           ell_c = T_oct  ell_p
//   M2L: 316 same-level offsets d in [-3,3]^3 \ [-1,1]^3 (classical 1-box
//        separation V list)                  ell   = T_d    mu
// Storage convention (per box, box width s, centre c, u = (x - c)/s):
//   P2M  mu  = sum_l q_l Rt(u_l)                   (plain sum of harmonic vectors)
//   M2P  phi = (1/s) sum_i w_i mu_i It_i(u)        (w = 1 for m = 0, 2 otherwise)
//   P2L  ell = sum_l q_l w_i It_i(u_l)
//   L2P  phi = (1/s) sum_i ell_i Rt_i(u)
#pragma once

#include <vector>

#include "harmonics.h"

namespace xrl {

constexpr int kNM2L = 316;

struct HostOperators {
    std::vector<double> m2m;   // [8][kNC][kNC]   out-major (row = output coefficient)
    std::vector<double> l2l;   // [8][kNC][kNC]
    std::vector<double> m2l;   // [316][kNC][kNC]
    int m2l_off[kNM2L][3];     // offset (target - source) in box widths
    int m2l_index[343];        // (dx+3)*49 + (dy+3)*7 + (dz+3) -> 0..315 or -1
};

// Build all operators for order kP in FP64.
void build_operators(HostOperators& ops);

// Octant index of a child: bit0 = +x half, bit1 = +y, bit2 = +z.
inline int octant(int bx, int by, int bz) { return bx | (by << 1) | (bz << 2); }

}  // namespace xrl
