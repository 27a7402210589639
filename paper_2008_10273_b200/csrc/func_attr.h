// Per-device kernel attributes.  cudaFuncSetAttribute applies to the current
// device only, so a process that launches on several GPUs must set them on
// each: this remembers (device, kernel, attribute) and sets each once.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <tuple>

#include "common.h"

namespace hivc {

inline void ensure_func_attr(const void* fn, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, int, int>> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) fail(HIVC_E_CUDA, "cudaGetDevice failed");
    const auto key = std::make_tuple(dev, fn, (int)attr, value);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(key)) return;
    const cudaError_t e = cudaFuncSetAttribute(fn, attr, value);
    if (e != cudaSuccess) fail(HIVC_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    done.insert(key);
}

}  // namespace hivc
