// Copy-engine facts on this B200 (development probe, not product code):
//  1. does a same-device D2D cudaMemcpyAsync need SMs? (launched while an
//     SM-hog kernel occupies every SM: if it completes before the hog ends,
//     it ran on a copy engine)
//  2. D2D copy bandwidth vs size and number of concurrent streams
//  3. cost of satisfied / unsatisfied cuStreamWaitValue32 on a copy stream
//  4. the CUDA runtime version
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ce_probe.cu -lcuda -o build/ce_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t err_ = (x);                                                           \
        if (err_ != cudaSuccess) {                                                      \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(err_)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__global__ void hog(long long cycles, int* flag) {
    extern __shared__ char sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {
        if (threadIdx.x == 0 && sm[0] == 42) flag[0] = 1;
    }
}

__global__ void bump(unsigned* p, unsigned v) { *p = v; }

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    printf("{\"device\": \"%s\", \"asyncEngineCount\": %d, \"sms\": %d,\n", prop.name,
           prop.asyncEngineCount, prop.multiProcessorCount);
    const size_t big = size_t(1) << 30;
    char *a, *b;
    CK(cudaMalloc(&a, big));
    CK(cudaMalloc(&b, big));
    CK(cudaMemset(a, 1, big));
    int* flag;
    CK(cudaMalloc(&flag, 4));
    cudaStream_t s_hog, s_cp[8];
    CK(cudaStreamCreateWithFlags(&s_hog, cudaStreamNonBlocking));
    for (auto& s : s_cp) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, e2, e3;
    for (auto* ev : {&e0, &e1, &e2, &e3}) CK(cudaEventCreate(ev));

    // 1. SM hog: 2 CTAs x 1024 threads x 100KB smem per SM -> no room for anything
    CK(cudaFuncSetAttribute(hog, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 << 10));
    const long long cycles = 20LL * 1000 * 1000;  // ~10 ms at ~2 GHz
    CK(cudaEventRecord(e0, s_hog));
    hog<<<prop.multiProcessorCount * 2, 1024, 110 << 10, s_hog>>>(cycles, flag);
    CK(cudaEventRecord(e1, s_hog));
    CK(cudaStreamWaitEvent(s_cp[0], e0, 0));
    CK(cudaMemcpyAsync(b, a, 256 << 20, cudaMemcpyDeviceToDevice, s_cp[0]));
    CK(cudaEventRecord(e2, s_cp[0]));
    CK(cudaDeviceSynchronize());
    float hog_ms, cp_ms;
    CK(cudaEventElapsedTime(&hog_ms, e0, e1));
    CK(cudaEventElapsedTime(&cp_ms, e0, e2));
    printf("\"hog_ms\": %.3f, \"d2d_256MiB_done_at_ms\": %.3f, \"d2d_uses_copy_engine\": %s,\n", hog_ms,
           cp_ms, cp_ms < 0.8 * hog_ms ? "true" : "false");

    // 2. bandwidth vs size and streams (one buffer pair split among streams)
    printf("\"d2d_bw_GBps\": {");
    bool first = true;
    for (size_t sz : {size_t(1) << 20, size_t(4) << 20, size_t(16) << 20, size_t(112) << 20,
                      size_t(512) << 20}) {
        for (int ns : {1, 2, 4, 8}) {
            float best = 1e30f;
            for (int it = 0; it < 5; ++it) {
                CK(cudaEventRecord(e0, s_cp[0]));
                for (int i = 1; i < ns; ++i) CK(cudaStreamWaitEvent(s_cp[i], e0, 0));
                const size_t part = sz / ns;
                for (int i = 0; i < ns; ++i)
                    CK(cudaMemcpyAsync(b + i * part, a + i * part, part, cudaMemcpyDeviceToDevice, s_cp[i]));
                for (int i = 1; i < ns; ++i) {
                    CK(cudaEventRecord(e3, s_cp[i]));
                    CK(cudaStreamWaitEvent(s_cp[0], e3, 0));
                }
                CK(cudaEventRecord(e1, s_cp[0]));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            printf("%s\"%zuMiB_x%d\": %.1f", first ? "" : ", ", sz >> 20, ns, sz / best / 1e6);
            first = false;
        }
    }
    printf("},\n");

    // 3. stream-memop wait cost: N satisfied waits + 4 KiB copies on one stream
    cuInit(0);
    unsigned* word;
    CK(cudaMalloc(&word, 4));
    CK(cudaMemset(word, 0, 4));
    for (int nwait : {0, 64, 256}) {
        CK(cudaEventRecord(e0, s_cp[0]));
        for (int i = 0; i < 256; ++i) {
            if (i < nwait)
                cuStreamWaitValue32((CUstream)s_cp[0], (CUdeviceptr)word, 0, CU_STREAM_WAIT_VALUE_GEQ);
            CK(cudaMemcpyAsync(b, a, 4096, cudaMemcpyDeviceToDevice, s_cp[0]));
        }
        CK(cudaEventRecord(e1, s_cp[0]));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("\"256_copies_4KiB_with_%d_satisfied_waits_us\": %.1f,\n", nwait, ms * 1e3);
    }
    // unsatisfied wait released by a kernel on another stream: wake-up latency
    {
        float tot = 0;
        for (int it = 0; it < 20; ++it) {
            CK(cudaMemset(word, 0, 4));
            CK(cudaDeviceSynchronize());
            cuStreamWaitValue32((CUstream)s_cp[0], (CUdeviceptr)word, it + 1, CU_STREAM_WAIT_VALUE_GEQ);
            CK(cudaEventRecord(e1, s_cp[0]));
            CK(cudaEventRecord(e0, s_hog));
            bump<<<1, 1, 0, s_hog>>>(word, it + 1);
            CK(cudaEventRecord(e2, s_hog));
            CK(cudaDeviceSynchronize());
            float ms;
            CK(cudaEventElapsedTime(&ms, e2, e1));
            tot += ms;
        }
        printf("\"wait_wakeup_after_kernel_write_us\": %.2f,\n", tot / 20 * 1e3);
    }
    // 4. runtime version
    printf("\"cuda_runtime_version\": %d}\n", CUDART_VERSION);
    return 0;
}
