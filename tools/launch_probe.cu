// Launch-overhead probe for the fused small-grid step (C1): how long does an (almost) empty
// kernel take between two CUDA events, as a plain 16-CTA grid, as a 16-CTA cluster
// (non-portable size) and as an 8-CTA cluster, with and without dynamic shared memory, directly
// launched and from a one-node CUDA graph. Also the cost of one cluster barrier and of a global
// write -> cluster barrier -> read round trip, measured on the device with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void empty_kernel(int *p) {
    extern __shared__ double s[];
    if (p && threadIdx.x == 1023) p[0] = (int)s[0];
}

__global__ void barrier_kernel(long long *out, int reps, double *buf) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < reps; ++i) cl.sync();
    long long t1 = clock64();
    // write -> barrier -> read (L2) round trips
    const int r = (int)cl.block_rank(), n = (int)cl.num_blocks();
    double acc = 0;
    for (int i = 0; i < reps; ++i) {
        buf[r * 256 + threadIdx.x] = acc + i;
        cl.sync();
        acc += __ldcg(buf + ((r + 1) % n) * 256 + threadIdx.x);
    }
    long long t2 = clock64();
    // DSMEM: write to the neighbour's shared memory -> barrier -> read locally
    __shared__ double sm[256];
    double *remote = cl.map_shared_rank(sm, (r + 1) % n);
    for (int i = 0; i < reps; ++i) {
        remote[threadIdx.x] = acc + i;
        cl.sync();
        acc += sm[threadIdx.x];
        cl.sync();
    }
    long long t3 = clock64();
    if (threadIdx.x == 0 && r == 0) {
        out[0] = (t1 - t0) / reps;
        out[1] = (t2 - t1) / reps;
        out[2] = (t3 - t2) / reps;
        out[3] = (long long)acc;
    }
}

struct Cfg { const char *name; int grid, cluster; size_t smem; };

static float time_launches(const Cfg &c, cudaStream_t st, int n, bool graph, int *dummy) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.cluster > 1 ? 1 : 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphExec_t ge = nullptr;
    if (graph) {
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        cudaLaunchKernelEx(&cfg, empty_kernel, dummy);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
    }
    // back-to-back
    for (int i = 0; i < 20; ++i) graph ? (void)cudaGraphLaunch(ge, st) : (void)cudaLaunchKernelEx(&cfg, empty_kernel, dummy);
    cudaEventRecord(e0, st);
    for (int i = 0; i < n; ++i) graph ? (void)cudaGraphLaunch(ge, st) : (void)cudaLaunchKernelEx(&cfg, empty_kernel, dummy);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ge) cudaGraphExecDestroy(ge);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms * 1000.f / n;
}

// one launch between two events, after a long kernel (the bench's situation: the host is ahead)
static float time_single(const Cfg &c, cudaStream_t st, int *dummy, double *big, size_t nbig) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.cluster > 1 ? 1 : 0;
    std::vector<float> v;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 60; ++i) {
        cudaMemsetAsync(big, i, nbig, st);
        cudaEventRecord(e0, st);
        cudaLaunchKernelEx(&cfg, empty_kernel, dummy);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 10) v.push_back(ms * 1000.f);
    }
    std::sort(v.begin(), v.end());
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return v[v.size() / 2];
}

int main() {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int *dummy;
    CK(cudaMalloc(&dummy, 64));
    double *big;
    const size_t nbig = 256u << 20;
    CK(cudaMalloc(&big, nbig));
    CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    Cfg cfgs[] = {{"grid16", 16, 1, 0},          {"grid16_smem48k", 16, 1, 48 << 10},
                  {"grid148", 148, 1, 0},        {"cluster16", 16, 16, 0},
                  {"cluster16_smem48k", 16, 16, 48 << 10}, {"cluster8", 8, 8, 0},
                  {"cluster8_smem48k", 8, 8, 48 << 10},    {"grid32_cluster2", 32, 2, 48 << 10}};
    for (const Cfg &c : cfgs) {
        const float b2b = time_launches(c, st, 1000, false, dummy);
        const float b2bg = time_launches(c, st, 1000, true, dummy);
        const float single = time_single(c, st, dummy, (double *)big, nbig);
        CK(cudaGetLastError());
        printf("{\"probe\": \"launch\", \"cfg\": \"%s\", \"back_to_back_us\": %.2f, \"graph_back_to_back_us\": %.2f, "
               "\"single_after_memset_us\": %.2f}\n", c.name, b2b, b2bg, single);
    }
    // barrier costs in cycles
    CK(cudaFuncSetAttribute(barrier_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    long long *d_out;
    double *buf;
    CK(cudaMalloc(&d_out, 4 * sizeof(long long)));
    CK(cudaMalloc(&buf, 16 * 256 * sizeof(double)));
    for (int cs : {8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, barrier_kernel, d_out, 200, buf));
        CK(cudaStreamSynchronize(st));
        long long h[4];
        CK(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost));
        printf("{\"probe\": \"cluster_sync\", \"cluster\": %d, \"barrier_cyc\": %lld, \"l2_write_barrier_read_cyc\": %lld, "
               "\"dsmem_write_barrier_read_barrier_cyc\": %lld}\n", cs, h[0], h[1], h[2]);
    }
    return 0;
}
