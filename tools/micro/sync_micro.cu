// Latency micro-benchmarks (single warp chains) for the warp/CTA/cluster
// primitives used by the cluster FPS exchange.  sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#define IT 2048

__global__ void k_redux(unsigned* out, long long* cyc) {
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) x = __reduce_max_sync(0xffffffffu, x + threadIdx.x) & 0xffff;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void k_shfl(unsigned* out, long long* cyc) {
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void k_ballot(unsigned* out, long long* cyc) {
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) x = __ballot_sync(0xffffffffu, (x >> (threadIdx.x & 7)) & 1) + threadIdx.x;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void k_lds(unsigned* out, long long* cyc) {
    __shared__ unsigned s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) x = s[x];
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void k_match(unsigned* out, long long* cyc) {
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) x = __match_any_sync(0xffffffffu, x & 7) + (x & 7);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void k_bar(unsigned* out, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < IT; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_cluster_bar(unsigned* out, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < IT / 8; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) * 8;
}
// ping-pong between CTA 0 and CTA 1 of a cluster via st.async + mbarrier
__global__ void k_pingpong(unsigned* out, long long* cyc) {
    __shared__ __align__(8) unsigned long long bar;
    __shared__ __align__(16) unsigned slot[4];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    const unsigned baddr = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(slot);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(baddr));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    const unsigned peer = r ^ 1;
    unsigned rs, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rs) : "r"(saddr), "r"(peer));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(baddr), "r"(peer));
    long long t0 = clock64();
    const int rounds = 256;
    for (int i = 0; i < rounds; ++i) {
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], 16;" ::"r"(baddr) : "memory");
        if ((i & 1) == (int)r) {
            if (threadIdx.x == 0)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%2, %2, %2, %2}, [%1];" ::"r"(rs), "r"(rb), "r"((unsigned)i) : "memory");
            // also wait for my own incoming message? no: one message per round, receiver waits
        }
        if ((i & 1) != (int)r) {
            asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"(baddr), "r"((unsigned)((i >> 1) & 1)) : "memory");
        } else {
            // sender: complete its own barrier phase locally with a dummy tx so parity stays aligned
            if (threadIdx.x == 0) asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], 16;" ::"r"(baddr) : "memory");
            asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n" ::"r"(baddr), "r"((unsigned)((i >> 1) & 1)) : "memory");
        }
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (threadIdx.x == 0 && r == 0) cyc[0] = (t1 - t0) * IT / rounds;
}

int main() {
    unsigned* out; long long* cyc; long long h;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    auto run = [&](const char* nm, void (*k)(unsigned*, long long*), int threads) {
        k<<<1, threads>>>(out, cyc); cudaDeviceSynchronize();
        k<<<1, threads>>>(out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.1f cycles/op\n", nm, (double)h / IT);
    };
    run("REDUX.max (dep chain)", k_redux, 32);
    run("SHFL.idx (dep chain)", k_shfl, 32);
    run("VOTE.ballot (dep chain)", k_ballot, 32);
    run("LDS (pointer chase)", k_lds, 32);
    run("MATCH.any (dep chain)", k_match, 32);
    run("__syncthreads 256 thr", k_bar, 256);
    run("__syncthreads 1024 thr", k_bar, 1024);
    for (int C : {2, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        if (C > 8) cudaFuncSetAttribute(k_cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchKernelEx(&cfg, k_cluster_bar, out, cyc); cudaDeviceSynchronize();
        cudaLaunchKernelEx(&cfg, k_cluster_bar, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("barrier.cluster C=%-2d          %.1f cycles/op  (%s)\n", C, (double)h / IT, cudaGetErrorString(cudaGetLastError()));
    }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2); cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_pingpong, out, cyc); cudaDeviceSynchronize();
        cudaLaunchKernelEx(&cfg, k_pingpong, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("st.async+mbarrier one-way     %.1f cycles  (%s)\n", (double)h / IT, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
