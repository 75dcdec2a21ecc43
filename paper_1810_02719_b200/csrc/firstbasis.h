// First-submesh basis (K9), see firstbasis.cu.
#pragma once

#include <cstdlib>

#include <stdint.h>

#include <algorithm>
#include <vector>

#include "engine.h"

namespace smg {

struct FirstBasisConfig {
    int dense_limit = 4096;
    int initial_iterations = 60;
    int power = 2;
    uint64_t seed = 1;
    int max_rounds = 12;
    double tol = 1e-10;  // subspace-angle bound; parity target 1e-8
    double shift_hint = 0.0;
};

struct FirstBasisReport {
    int iterations = 0;
    int rounds = 0;
    double bound = 0.0;
    bool cold = false;
};

// Columns of the first-basis subspace: c plus max(16, c/2) guard columns,
// capped at the 480-column limit of the cluster Jacobi (16 CTAs x 2 blocks of 15).
constexpr int kFirstBasisMaxCols = 480;
inline int first_basis_width(int n, int c) {
    static const int div = std::getenv("SMG_FB_GUARD") ? std::max(1, std::atoi(std::getenv("SMG_FB_GUARD"))) : 6;
    const int want = round_up(c + std::max(16, c / div), 8);
    return std::min(n, std::max(c, std::min(kFirstBasisMaxCols, want)));
}

std::vector<double> gaussian_block_colmajor(int rows, int cols, uint64_t seed);
// Writes the first basis (n x c, row-major, unsigned columns) into ws.U for every
// batch entry b, whose tile is tile0 + b * tstride.
FirstBasisReport first_basis(const StepCtx& cx, Workspace& ws, const TileSet& ts, int tile0, int tstride, int c,
                             const FirstBasisConfig& cfg, const FactorSet* op_factor);

}  // namespace smg
