// Device-side cost of an (almost) empty persistent kernel as a function of
// dynamic shared memory and block size (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int *out) {
    extern __shared__ int dsm[];
    __shared__ int sm[1];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (sm[0] == -1) out[0] = 1;
}
int main() {
    int *out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int smems[] = {0, 48 * 1024, 100 * 1024, 160 * 1024, 222 * 1024};
    int threads[] = {256, 608, 1024};
    for (int sm : smems) {
        cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        for (int th : threads) {
            for (int w = 0; w < 3; ++w) empty_k<<<144, th, sm>>>(out);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int i = 0; i < 200; ++i) empty_k<<<144, th, sm>>>(out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("smem %6d B  threads %4d : %6.2f us per launch (back-to-back) %s\n", sm, th, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
