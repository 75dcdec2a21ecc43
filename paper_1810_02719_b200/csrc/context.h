// Opaque handle definitions shared by the C-ABI translation units.
#pragma once

#include <string>

#include "engine.h"

struct smg_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string error;
};

struct smg_operator {
    smg::TileSet ts;
    smg::FactorSet fs;
    int n = 0, z = 1;
    double delta = 0.0;
};
