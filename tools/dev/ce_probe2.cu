// Which same-device copy paths run on a copy engine (no SMs)? Each candidate
// is issued while an SM-hog kernel fills every SM for ~10 ms; a copy that
// finishes well before the hog ran on a copy engine. Development probe.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t err_ = (x);                                                            \
        if (err_ != cudaSuccess) {                                                         \
            printf("\"error\": \"%s line %d: %s\"}\n", #x, __LINE__, cudaGetErrorString(err_)); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void hog(long long cycles) {
    extern __shared__ char sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {
        if (sm[threadIdx.x] == 42) sm[0] = 1;
    }
}

static cudaStream_t s_hog, s_cp;
static cudaEvent_t e0, e1, e2;

template <class F>
int under_hog(const char* name, F copy, size_t bytes) {
    const long long cycles = 20LL * 1000 * 1000;
    CK(cudaEventRecord(e0, s_hog));
    hog<<<148 * 2, 1024, 110 << 10, s_hog>>>(cycles);
    CK(cudaEventRecord(e1, s_hog));
    CK(cudaStreamWaitEvent(s_cp, e0, 0));
    CK(copy());
    CK(cudaEventRecord(e2, s_cp));
    CK(cudaDeviceSynchronize());
    float hog_ms, cp_ms;
    CK(cudaEventElapsedTime(&hog_ms, e0, e1));
    CK(cudaEventElapsedTime(&cp_ms, e0, e2));
    // bandwidth without the hog
    CK(cudaEventRecord(e0, s_cp));
    CK(copy());
    CK(cudaEventRecord(e2, s_cp));
    CK(cudaEventSynchronize(e2));
    float alone;
    CK(cudaEventElapsedTime(&alone, e0, e2));
    printf("\"%s\": {\"hog_ms\": %.3f, \"done_ms\": %.3f, \"copy_engine\": %s, \"alone_GBps\": %.1f},\n",
           name, hog_ms, cp_ms, cp_ms < 0.7 * hog_ms ? "true" : "false", bytes / alone / 1e6);
    return 0;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const size_t n = size_t(256) << 20;
    char *a, *b, *h;
    CK(cudaMalloc(&a, n));
    CK(cudaMalloc(&b, n));
    CK(cudaHostAlloc(&h, n, cudaHostAllocDefault));
    CK(cudaStreamCreateWithFlags(&s_hog, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s_cp, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    CK(cudaFuncSetAttribute(hog, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 << 10));
    printf("{");
    under_hog("memcpyAsync_d2d", [&] { return cudaMemcpyAsync(b, a, n, cudaMemcpyDeviceToDevice, s_cp); }, n);
    under_hog("memcpyPeerAsync_same_dev", [&] { return cudaMemcpyPeerAsync(b, 0, a, 0, n, s_cp); }, n);
    under_hog("memcpy2DAsync_d2d", [&] {
        return cudaMemcpy2DAsync(b, 1 << 20, a, 1 << 20, 1 << 20, n >> 20, cudaMemcpyDeviceToDevice, s_cp);
    }, n);
    under_hog("memcpyAsync_d2h_pinned", [&] { return cudaMemcpyAsync(h, a, n, cudaMemcpyDeviceToHost, s_cp); }, n);
    under_hog("memcpyAsync_h2d_pinned", [&] { return cudaMemcpyAsync(a, h, n, cudaMemcpyHostToDevice, s_cp); }, n);
    printf("\"done\": true}\n");
    return 0;
}
