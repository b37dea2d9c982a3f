// Per-iteration floor of the FPS exchange skeleton inside one CTA (sm_100a):
// warp argmax -> record in smem -> barrier -> leader reduce -> broadcast.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o iter_micro iter_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 2000;

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// mode 0: __syncthreads x2, every warp reduces the records itself
// mode 1: named barriers, leader reduces + broadcasts
// mode 2: one warp alone (no barrier): LDS -> REDUX -> STS -> LDS
// mode 3: __syncthreads only (two per iteration), no reductions
template <int MODE>
__global__ void k(unsigned* out, long long* cyc, int nthreads) {
    __shared__ unsigned rec[32];
    __shared__ unsigned win;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned x = threadIdx.x * 2654435761u;
    if (threadIdx.x == 0) win = 1;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) {
        const unsigned s = win;
        x = x * 1664525u + s;
        if (MODE == 2) {
            if (warp != 0) break;
            const unsigned m = __reduce_max_sync(0xffffffffu, x >> 8);
            if (lane == 0) rec[0] = m;
            __syncwarp();
            if (lane == 0) win = rec[0] & 0xffff;
            __syncwarp();
            continue;
        }
        if (MODE == 3) {
            __syncthreads();
            if (threadIdx.x == 0) win = x & 0xff;
            __syncthreads();
            continue;
        }
        const unsigned m = __reduce_max_sync(0xffffffffu, x >> 8);
        if (lane == 0) rec[warp] = m;
        if (MODE == 0) {
            __syncthreads();
            const unsigned r = lane < nw ? rec[lane] : 0u;
            const unsigned g = __reduce_max_sync(0xffffffffu, r);
            __syncthreads();
            if (threadIdx.x == 0) win = g & 0xffff;
            __syncthreads();
        } else {
            if (warp == nw - 1) {
                nb_sync(1, blockDim.x);
                const unsigned r = lane < nw ? rec[lane] : 0u;
                const unsigned g = __reduce_max_sync(0xffffffffu, r);
                if (lane == 0) win = g & 0xffff;
                nb_arrive(2, blockDim.x);
            } else {
                nb_arrive(1, blockDim.x);
                nb_sync(2, blockDim.x);
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

template <int MODE>
void run(const char* name, int threads) {
    unsigned* o;
    long long* c;
    cudaMalloc(&o, 4);
    cudaMalloc(&c, 8);
    k<MODE><<<1, threads>>>(o, c, threads);
    k<MODE><<<1, threads>>>(o, c, threads);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-44s threads=%4d: %7.1f cycles/iter\n", name, threads, (double)h / IT);
    cudaFree(o);
    cudaFree(c);
}

int main() {
    for (int t : {32, 128, 256, 512, 1024}) {
        run<0>("syncthreads x3, all warps reduce", t);
        run<1>("named barriers, leader reduce + broadcast", t);
        run<3>("syncthreads x2 only", t);
    }
    run<2>("one warp: LDS-REDUX-STS-LDS", 32);
    return 0;
}
