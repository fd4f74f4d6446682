// common.cuh -- shared constants, geometry / tile / sinogram-view records
// (part of kernels.cuh; notation and layouts: see kernels.cuh and DESIGN.md)
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>
#include <type_traits>

namespace lt {

namespace cg = cooperative_groups;

constexpr int PADL = 4;           // left zero padding of padded tile rows
constexpr int PADR = 4;           // right zero padding
constexpr float MAGICF = 12582912.0f;   // 1.5 * 2^23: x + MAGICF rounds x to an integer in the low mantissa bits
constexpr int MAGICI = 0x4B400000;

struct AngF {       // per-angle constants (fp32), 32 B
    float cs, sn;   // cos, sin
    float invc;     // 1/c, c = max(|cos|,|sin|)
    float ic2;      // 1/c^2
    float K;        // 1/c - 0.5/c^2  (hat weights in the magic-floor form)
    float A, B;     // Joseph marching: pos(w, l) = Lc + (w - tau_c) A + (l - Lc) B
    int col;        // 1 = column-driven (|sin| > |cos|): march columns on the transposed image
};

struct TileT {      // per tile, tile-local coordinates
    int row0, col0;           // global coords of tile pixel (0,0) (negative if clipped)
    int vr0, vr1, vc0, vc1;   // valid rectangle (inside the grid), half-open
    int pad0, pad1;
};

struct Geo {
    int n, na, nd;
    const AngF* ang;
    const double* cs64;
    const double* sn64;
    const double* A64;
    const double* B64;
};

struct Tiles {
    int T, TP, Wwin, ntiles;
    const TileT* tile;
    const int* d0;          // [tile][na] window start (global bin index)
    const double* tauc;     // [tile][na] bin coordinate of the tile centre relative to d0
};

struct SinoView {           // element (tile r, angle a, window bin w)
    const float* base;
    long long tile_stride;  // elements between tiles (0 = shared sinogram)
    int row_stride;         // elements between angles
    int use_d0;             // 1: index = d0[r][a] + w (full sinogram); 0: index = w (window sinogram)
    int len;                // valid index range [0, len)
};

__device__ __forceinline__ float sv_fetch(const SinoView& s, const int* d0, int na, int r, int a, int w) {
    const int idx = (s.use_d0 ? __ldg(d0 + r * na + a) : 0) + w;
    if (idx < 0 || idx >= s.len) return 0.f;
    return __ldg(s.base + (long long)r * s.tile_stride + (long long)a * s.row_stride + idx);
}

}  // namespace lt
