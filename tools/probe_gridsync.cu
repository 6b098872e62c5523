// probe_gridsync.cu — cost of cooperative grid.sync() vs grid size on this GPU.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_gridsync tools/probe_gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = n;
}
// hand-rolled: one flag word per phase, arrive with red.release, poll with ld.acquire
__device__ unsigned int g_bar;
__global__ void k_sync2(int n, int* out) {
    unsigned int target = 0;
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        target += gridDim.x;
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&g_bar) : "memory");
            unsigned int v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_bar) : "memory");
            } while ((int)(v - target) < 0);
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = n;
}
int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int cfg[][2] = {{592, 256}, {296, 512}, {148, 1024}, {148, 256}};
    for (auto& c : cfg) {
        for (int n : {0, 200}) {
            for (int coop = 0; coop < 2; ++coop) {
                if (!coop && n) continue;  // grid.sync needs a cooperative launch
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    void* args[] = {&n, &d};
                    cudaEventRecord(a);
                    if (coop)
                        cudaLaunchCooperativeKernel((void*)k_sync, c[0], c[1], args, 0, 0);
                    else
                        cudaLaunchKernel((void*)k_sync, c[0], c[1], args, 0, 0);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("%s grid %d x %d, %d syncs: %.1f us total (%s)\n", coop ? "cooperative" : "plain      ", c[0], c[1], n,
                       best * 1000, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
}
