// pf_bvh.cuh -- the linear BVH over the cells' bounding balls, shared by the
// Čech graph builder (pf_cech.cu, NEXT-3) and the adjacency-walk tracer's gap
// jumps (pf_trace.cu, NEXT-4).  30-bit Morton codes of the sites sorted by the
// K4 radix sort, Karras' radix tree, bottom-up box refit (pf_cech.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_internal.cuh"

namespace pf {

struct Box {
    float lo[3], hi[3];
};

// Node encoding: children (idx << 1) | is_leaf; internal node 0 is the root
// (n > 1); leaf k holds ball order[k] with box bleaf[k].
struct BallBVH {
    DevBuf keys, keys_alt, vals, vals_alt, bb, left, right, pint, pleaf, bint, bleaf, arrive;
    const uint32_t *order = nullptr;
    int64_t n = 0;
    void release()
    {
        DevBuf *b[] = {&keys, &keys_alt, &vals, &vals_alt, &bb, &left, &right, &pint, &pleaf,
                       &bint, &bleaf, &arrive};
        for (auto *x : b) x->release();
        order = nullptr;
        n = 0;
    }
};

// Builds the BVH of the N balls (sites f32[N,3], radii f32[N], device) on `st`
// (no host sync); `scratch` supplies the sort workspaces and the launch counter.
cudaError_t build_ball_bvh(pf_scene *scratch, BallBVH &B, int64_t N, const float *sites,
                           const float *radii, cudaStream_t st);

}  // namespace pf
