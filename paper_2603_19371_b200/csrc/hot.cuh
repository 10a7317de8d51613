// hot.cuh -- shared machinery of the pipelined z-marching hot kernels.
//
// Every hot kernel owns a 32 x 8 column of output voxels and a chunk of z
// planes.  Per input plane it needs an (32 + 2H) x (8 + 2H) halo tile; each
// of the 256 threads owns at most two tile items, whose in-plane positions
// and global offsets are computed once (Items) and reused for every plane.
// Plane inputs are software-pipelined: dense loads run two planes ahead and
// data-dependent gathers one plane ahead of the plane being filtered, so HBM
// and L2 latency overlap the shared-memory filter passes.
#pragma once

#include "common.cuh"

namespace wlm {
namespace hot {

constexpr int TX = 32;
constexpr int TY = 8;
constexpr int NT = TX * TY;

template <int H>
struct Items {
    static constexpr int IW = TX + 2 * H, IH = TY + 2 * H, NI = IW * IH;
    static constexpr int SLOTS = (NI + NT - 1) / NT;
    int sidx[SLOTS];   // smem index iy * IW + ix (-1: no item)
    int gx[SLOTS], gy[SLOTS];
    int goff[SLOTS];   // gx + nx * gy, or -1 when outside the x/y extent
    __device__ __forceinline__ void init(int x0, int y0, int nx, int ny) {
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int idx = threadIdx.x + s * NT;
            if (idx < NI) {
                const int ix = idx % IW, iy = idx / IW;
                sidx[s] = idx;
                gx[s] = x0 - H + ix;
                gy[s] = y0 - H + iy;
                goff[s] = (gx[s] >= 0 && gx[s] < nx && gy[s] >= 0 && gy[s] < ny) ? gx[s] + nx * gy[s] : -1;
            } else {
                sidx[s] = -1;
                gx[s] = gy[s] = 0;
                goff[s] = -1;
            }
        }
    }
};

// fp64 rsqrt with one Newton step on top of the hardware estimate path that
// CUDA's rsqrt(double) already refines (kept as a named helper for clarity).
__device__ __forceinline__ double rsqrt_d(double v) { return rsqrt(v); }

}  // namespace hot
}  // namespace wlm
