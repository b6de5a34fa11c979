// Shared host-side helpers of the C ABI translation units (capi.cpp, dist.cpp, gmres.cpp): error
// mapping to the STIGA_* status codes (std::invalid_argument -> STIGA_INVALID_ARGUMENT, device
// failure -> STIGA_CUDA, any other std::exception -> STIGA_NUMERICAL), device guards and owned
// device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/linalg.hpp"
#include "stiga_gpu.h"

namespace stiga {
void set_last_error(const std::string& msg);  // capi.cpp: thread-local message behind stiga_last_error()

namespace capi {

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs f and maps its exception (if any) to a status code + the thread's last-error message.
template <typename F>
int guarded(F&& f) {
    try {
        f();
        set_last_error("");
        return STIGA_OK;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return STIGA_INVALID_ARGUMENT;
    } catch (const CudaFailure& e) {
        set_last_error(e.what());
        return STIGA_CUDA;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return STIGA_NUMERICAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return STIGA_NUMERICAL;
    }
}

inline void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

// Scoped device selection (restores the caller's current device).
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        ck(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Owned cudaMalloc'd double buffer (a cudaMalloc base pointer, so it can be exported by CUDA IPC).
struct DBuf {
    double* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        if (count) ck(cudaMalloc(&p, count * sizeof(double)), "cudaMalloc");
    }
    void ensure(size_t count) {
        if (!p || n < count) alloc(count);
    }
    void upload(const std::vector<double>& h) {
        alloc(h.size());
        if (!h.empty()) ck(cudaMemcpy(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
    }
};

inline DenseMatrix from_colmajor(const double* a, int n) {
    DenseMatrix m(n, n);
    std::memcpy(m.a.data(), a, sizeof(double) * n * static_cast<size_t>(n));
    return m;
}

// Row-major, zero-padded (Mp x Kp) copy of J, with J(i,j) = transpose ? U(j,i) : U(i,j).
inline std::vector<double> pad_factor(const DenseMatrix& U, bool transpose, int Mp, int Kp) {
    std::vector<double> out(static_cast<size_t>(Mp) * Kp, 0.0);
    const Index rows = transpose ? U.cols : U.rows;
    const Index cols = transpose ? U.rows : U.cols;
    if (rows > Mp || cols > Kp || Mp < 1)
        throw std::runtime_error("internal: no kernel tiling for a factor of size " + std::to_string(rows));
    for (Index i = 0; i < rows; ++i)
        for (Index j = 0; j < cols; ++j) out[i * Kp + j] = transpose ? U(j, i) : U(i, j);
    return out;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace capi
}  // namespace stiga
