// Driver-API entry points resolved at run time through the runtime's
// cudaGetDriverEntryPoint, so libc3cuda.so has no link-time dependency on
// libcuda.so.1: it loads (and reports "no device") on a machine without a
// GPU driver, which is how the CPU test suite checks its exported ABI.
#include <cuda_runtime.h>

#include "c3cuda_internal.hpp"

namespace c3k {

namespace {
template <class F>
void resolve(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        fn = reinterpret_cast<F>(p);
    else
        fn = nullptr;
}
}  // namespace

const Driver& drv() {
    static const Driver d = [] {
        Driver x{};
        resolve("cuGetErrorName", x.GetErrorName);
        resolve("cuInit", x.Init);
        resolve("cuDeviceGet", x.DeviceGet);
        resolve("cuDeviceGetDevResource", x.DeviceGetDevResource);
        resolve("cuDevSmResourceSplitByCount", x.DevSmResourceSplitByCount);
        resolve("cuDevResourceGenerateDesc", x.DevResourceGenerateDesc);
        resolve("cuGreenCtxCreate", x.GreenCtxCreate);
        resolve("cuGreenCtxDestroy", x.GreenCtxDestroy);
        resolve("cuGreenCtxStreamCreate", x.GreenCtxStreamCreate);
        resolve("cuStreamDestroy", x.StreamDestroy);
        resolve("cuStreamWriteValue32", x.StreamWriteValue32);
        resolve("cuStreamWaitValue32", x.StreamWaitValue32);
        resolve("cuTensorMapEncodeTiled", x.TensorMapEncodeTiled);
        return x;
    }();
    return d;
}

}  // namespace c3k
