// csr_fill.cu -- drop-in csr_fill (/root/reference/pkg/src/pointsample/_kernels.py:164-185)
// on the device.
//
// The reference scatters the undirected edges (ei[e], ej[e], ed[e]) of
// excl_collect into both rows in emission order, self first: row r holds
// r, then -- for every edge e touching r, e ascending -- the other endpoint.
// Here: the 2M directed half-edges are keyed by their row and stably radix
// sorted (CUB), which orders each row's half-edges by e; a half-edge at
// sorted position q of row r lands at indptr[r] + 1 + (q - (indptr[r] - r)),
// because the sorted array holds exactly deg(r') = indptr[r'+1] - indptr[r'] - 1
// half-edges of every earlier row r'.  Self entries are written separately.
// Bit-identical to the reference for any indptr that matches the degrees.

#include <cub/device/device_radix_sort.cuh>

#include <cstdint>

#include "ps_internal.h"

namespace ps {

namespace {

__global__ void halfedge_keys_kernel(const int32_t* __restrict__ ei, const int32_t* __restrict__ ej, int64_t M,
                                     uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 2 * M; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t >> 1;
        keys[t] = (uint32_t)((t & 1) ? ej[e] : ei[e]);
        vals[t] = (uint32_t)t;
    }
}

__global__ void csr_place_kernel(const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                                 const double* __restrict__ ed, int64_t M, const uint32_t* __restrict__ keys,
                                 const uint32_t* __restrict__ vals, const int64_t* __restrict__ indptr, int64_t N,
                                 int64_t* __restrict__ out_idx, double* __restrict__ out_d2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += stride) {
        out_idx[indptr[r]] = r;  // self first
        out_d2[indptr[r]] = 0.0;
    }
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < 2 * M; q += stride) {
        const int64_t r = keys[q];
        const uint32_t t = vals[q];
        const int64_t e = t >> 1;
        const int64_t slot = indptr[r] + 1 + (q - (indptr[r] - r));
        out_idx[slot] = (t & 1) ? ei[e] : ej[e];
        out_d2[slot] = ed[e];
    }
}

}  // namespace

size_t csr_fill_ws_bytes(int64_t M, int64_t N) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(2 * M), 0,
                                    N > 1 ? 32 - __builtin_clz((unsigned)(N - 1)) : 1);
    const size_t arr = (sizeof(uint32_t) * 2 * (size_t)M + 255) & ~size_t(255);
    return 4 * arr + ((temp + 255) & ~size_t(255));
}

cudaError_t launch_csr_fill(const int32_t* ei, const int32_t* ej, const double* ed, int64_t M, const int64_t* indptr,
                            int64_t N, int64_t* out_idx, double* out_d2, void* work, size_t work_bytes,
                            cudaStream_t s) {
    const size_t arr = (sizeof(uint32_t) * 2 * (size_t)M + 255) & ~size_t(255);
    unsigned char* w = static_cast<unsigned char*>(work);
    uint32_t* k_in = reinterpret_cast<uint32_t*>(w);
    uint32_t* v_in = reinterpret_cast<uint32_t*>(w + arr);
    uint32_t* k_out = reinterpret_cast<uint32_t*>(w + 2 * arr);
    uint32_t* v_out = reinterpret_cast<uint32_t*>(w + 3 * arr);
    void* temp = w + 4 * arr;
    size_t temp_bytes = work_bytes - 4 * arr;
    const unsigned g = (unsigned)std::min<int64_t>(148 * 16, (2 * M + N + 255) / 256 + 1);
    if (M > 0) {
        halfedge_keys_kernel<<<g, 256, 0, s>>>(ei, ej, M, k_in, v_in);
        const int bits = N > 1 ? 32 - __builtin_clz((unsigned)(N - 1)) : 1;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, (int)(2 * M), 0,
                                                        bits, s);
        if (e != cudaSuccess) return e;
    }
    csr_place_kernel<<<g, 256, 0, s>>>(ei, ej, ed, M, k_out, v_out, indptr, N, out_idx, out_d2);
    return cudaGetLastError();
}

}  // namespace ps
