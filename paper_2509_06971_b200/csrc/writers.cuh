// writers.cuh -- the reference's output writers from device buffers
// (field_io.cpp:29-126, engine.cpp:145-190).
//
// A field in HBM (padded rows, see Geo) becomes the exact bytes the reference
// writes: every value through "%.17g" (g17.cuh) followed by one separator byte
// ('\n' in a VTK array, ',' or '\n' at the end of an x row in a CSV field).  Two
// passes over blocks of TB consecutive values: (1) the byte count of every block,
// (2) after an exclusive scan of those counts, each block formats its values
// again into shared memory, compacts them with a block scan and stores its
// contiguous slice of the text with coalesced byte stores.  The host only adds
// the header lines (as the reference does, with snprintf) and writes the bytes.
// PGM (2D): the finite minimum / maximum with the reference's tie rule (the first
// of equal values in node order, so -0.0 and 0.0 are told apart as it does), then
// one byte per node, rows top-down.
#pragma once

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "g17.cuh"

namespace petto_b200 {
namespace wr {

constexpr int TB = 256;    // values per block
constexpr int MAXB = 25;   // bytes of one value (24) + its separator

// Field accessor: value i (node order x-fastest) of an nx x ny x nz block whose
// rows have pitch px and whose planes have stride plane (elements).
struct Src {
    const double* base;
    int nx, ny;
    long long px, plane, n;
};

__device__ __forceinline__ double value_at(const Src& s, long long i) {
    const long long r = i / s.nx;
    const int x = (int)(i - r * s.nx);
    const long long z = r / s.ny;
    const int y = (int)(r - z * s.ny);
    return s.base[z * s.plane + (long long)y * s.px + x];
}

// sep_mode 0: '\n' after every value (VTK); 1: ',' inside an x row, '\n' at its end (CSV)
__device__ __forceinline__ char separator(const Src& s, long long i, int sep_mode) {
    return (sep_mode == 0 || (i + 1) % s.nx == 0) ? '\n' : ',';
}

__global__ void __launch_bounds__(TB) k_block_bytes(Src s, long long i0, long long n, long long* block_bytes) {
    const long long i = i0 + (long long)blockIdx.x * TB + threadIdx.x;
    int len = 0;
    if (i < i0 + n) {
        char buf[MAXB];
        len = g17::format(value_at(s, i), buf) + 1;
    }
    // block sum (fixed order)
    __shared__ int part[TB / 32];
    for (int o = 16; o > 0; o >>= 1) len += __shfl_down_sync(0xffffffffu, len, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = len;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < TB / 32; ++w) t += part[w];
        block_bytes[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(TB) k_block_write(Src s, long long i0, long long n, int sep_mode,
                                                    const long long* block_off, char* out) {
    using Scan = cub::BlockScan<int, TB>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ char text[TB * MAXB];
    __shared__ int total;
    const long long i = i0 + (long long)blockIdx.x * TB + threadIdx.x;
    char buf[MAXB];
    int len = 0;
    if (i < i0 + n) {
        len = g17::format(value_at(s, i), buf);
        buf[len++] = separator(s, i, sep_mode);
    }
    int off = 0, sum = 0;
    Scan(tmp).ExclusiveSum(len, off, sum);
    for (int b = 0; b < len; ++b) text[off + b] = buf[b];
    if (threadIdx.x == 0) total = sum;
    __syncthreads();
    char* dst = out + block_off[blockIdx.x];
    for (int b = threadIdx.x; b < total; b += TB) dst[b] = text[b];
}

// ------------------------------------------------------------------ PGM
struct MinMax {
    double lo, hi;
    long long ilo, ihi;  // node index of lo / hi (LLONG_MAX: none yet)
};

// lo: the smallest finite value, the first in node order among equal ones
// (std::min keeps lo unless v < lo, field_io.cpp:76-80); hi likewise
__device__ __forceinline__ void mm_merge(MinMax& a, const MinMax& b) {
    if (b.ilo != 0x7fffffffffffffffLL) {
        if (b.lo < a.lo || (!(a.lo < b.lo) && b.ilo < a.ilo) || a.ilo == 0x7fffffffffffffffLL) {
            a.lo = b.lo;
            a.ilo = b.ilo;
        }
    }
    if (b.ihi != 0x7fffffffffffffffLL) {
        if (a.hi < b.hi || (!(b.hi < a.hi) && b.ihi < a.ihi) || a.ihi == 0x7fffffffffffffffLL) {
            a.hi = b.hi;
            a.ihi = b.ihi;
        }
    }
}

__global__ void __launch_bounds__(TB) k_minmax(Src s, MinMax* partial) {
    MinMax a{0.0, 0.0, 0x7fffffffffffffffLL, 0x7fffffffffffffffLL};
    for (long long i = (long long)blockIdx.x * TB + threadIdx.x; i < s.n; i += (long long)gridDim.x * TB) {
        const double v = value_at(s, i);
        if (!isfinite(v)) continue;
        MinMax b{v, v, i, i};
        mm_merge(a, b);
    }
    __shared__ MinMax sh[TB];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int o = TB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) mm_merge(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_minmax_final(MinMax* partial, int n) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    MinMax a = partial[0];
    for (int b = 1; b < n; ++b) mm_merge(a, partial[b]);
    partial[0] = a;
}

// one byte per node, image rows top-down (field_io.cpp:86-95)
__global__ void k_pgm_bytes(Src s, const MinMax* mm, unsigned char* out) {
    const bool any = mm->ilo != 0x7fffffffffffffffLL;
    const double lo = any ? mm->lo : 0.0, hi = any ? mm->hi : 0.0;
    const double span = hi > lo ? hi - lo : 1.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < s.n;
         i += (long long)gridDim.x * blockDim.x) {
        const double raw = value_at(s, i);
        const double v = isfinite(raw) ? __ddiv_rn(__dsub_rn(raw, lo), span) : 0.0;
        const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        const long long x = i % s.nx, y = i / s.nx;
        out[(s.ny - 1 - y) * s.nx + x] = (unsigned char)llround(__dmul_rn(255.0, c));
    }
}

}  // namespace wr
}  // namespace petto_b200
