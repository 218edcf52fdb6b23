// Host tableau of the library (see tableau.cpp).  Passed to every kernel BY
// VALUE as a launch parameter (kernel-parameter constant bank: uniform operands,
// no global __constant__ state shared between contexts).
#pragma once
#include <cstddef>

namespace irk {

struct Tableau {
    double c[8];      // c~_i
    double b[8];      // b~_i
    double mu[8][8];  // mu~_ij (symplectic rounding)
    double nu[8][8];  // nu~_ij (extrapolation, reading R-3)
    double hb[8];     // fl(h * b~_j)
};

int build_tableau(double h, Tableau *T, char *err, size_t errlen);

}  // namespace irk
