// F1: segmentation on the GPU -- partition_mesh (partition.hpp:84-159),
// expand_overlaps (:205-253), order_submeshes (:258-307), i.e. segment_mesh
// (pipeline.hpp:131-138), bit-exact with the reference's tie rules.
#pragma once

#include <cstdint>
#include <vector>

#include "engine.h"

namespace smg {

// Vertex graph of a mesh on the device (EdgeSet neighbour lists as CSR).
struct GraphDev {
    int n = 0;
    const int32_t* offs = nullptr;
    const int32_t* cols = nullptr;
};

// Segmentation built on the device: per-vertex part id, the k sorted member
// lists of n_d vertices (k x n_d, row = submesh id) and the visiting order.
struct DeviceSegmentation {
    int k = 0, n_d = 0;
    DBuf<int32_t> assignment, offsets, members;
    std::vector<int32_t> offsets_h, sequence_h;
};

// partition_mesh: farthest-point seeds (hop-distance BFS), then the greedy
// smallest-part growth.  Throws Failure(2) with the reference's texts.
void partition_mesh_dev(const GraphDev& g, int k, uint64_t seed, int32_t* assignment, cudaStream_t st);
// expand_overlaps: every part grown by BFS rings to n_d = floor(growth * max
// part size); members (k x n_d, sorted per row) allocated here.  Returns n_d.
int expand_overlaps_dev(const GraphDev& g, const int32_t* assignment, int k, double growth, DBuf<int32_t>& members,
                        cudaStream_t st);
// order_submeshes over k equal-sized sorted member lists (k x n_d).
std::vector<int32_t> order_submeshes_dev(const int32_t* members, int k, int n_d, int n, uint64_t seed,
                                         cudaStream_t st);
// segment_mesh = the three above.
void segment_mesh_dev(const GraphDev& g, int k, double growth, uint64_t seed, DeviceSegmentation& out,
                      cudaStream_t st);

}  // namespace smg
