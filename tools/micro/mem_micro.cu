// Dependent-load latency through L1/L2 and cluster barrier cost (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mem_micro mem_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 4096;

// MODE 0: ld.global (default caching); 1: ld.global.cg (L2 only); 2: ld.relaxed.gpu
template <int MODE>
__global__ void chase(const int* __restrict__ nxt, long long* cyc, int* out) {
    int x = threadIdx.x * 97;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) {
        if (MODE == 0) x = nxt[x];
        else if (MODE == 1) x = __ldcg(nxt + x);
        else asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(nxt + x) : "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

__global__ void cluster_bar(long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    const int n = 1 << 22;  // 16 MB: L2 resident, larger than L1
    int* h = new int[n];
    // random cycle
    uint64_t s = 12345;
    int* perm = new int[n];
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = n - 1; i > 0; --i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        int j = (int)((s >> 33) % (uint64_t)(i + 1));
        int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    for (int i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
    int* d;
    long long* c;
    int* o;
    cudaMalloc(&d, sizeof(int) * n);
    cudaMalloc(&c, 8);
    cudaMalloc(&o, 4);
    cudaMemcpy(d, h, sizeof(int) * n, cudaMemcpyHostToDevice);
    long long hc;
    for (int rep = 0; rep < 2; ++rep) {
        chase<0><<<1, 1>>>(d, c, o);
        cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("ld.global chase (16MB, 1 thread):        %.1f cycles/load\n", (double)hc / IT);
        chase<1><<<1, 1>>>(d, c, o);
        cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("ld.global.cg chase:                      %.1f cycles/load\n", (double)hc / IT);
        chase<2><<<1, 1>>>(d, c, o);
        cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("ld.relaxed.gpu chase:                    %.1f cycles/load\n", (double)hc / IT);
        chase<1><<<148, 1024>>>(d, c, o);
        cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("ld.global.cg chase, 148x1024 threads:    %.1f cycles/load\n", (double)hc / IT);
    }
    for (int C : {2, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C, 1, 1);
        cfg.blockDim = dim3(1024, 1, 1);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (C > 8) cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchKernelEx(&cfg, cluster_bar, c);
        cudaLaunchKernelEx(&cfg, cluster_bar, c);
        cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        printf("barrier.cluster C=%2d x 1024 threads:       %.1f cycles/barrier (%s)\n", C, (double)hc / 256,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
