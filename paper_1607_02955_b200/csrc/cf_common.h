// Shared helpers for the cfcent_b200 library: error reporting and CUDA checks.
#pragma once
#include <cstdio>
#include <stdexcept>
#include <string>

namespace cf {

void set_error(const std::string& msg);

struct CfError : std::runtime_error {
    int code;
    double best_residual;
    CfError(int c, const std::string& m, double br = 0.0)
        : std::runtime_error(m), code(c), best_residual(br) {}
};

}  // namespace cf

#define CF_API_BEGIN try {
#define CF_API_END                                                   \
    }                                                                \
    catch (const cf::CfError& e) {                                   \
        cf::set_error(e.what());                                     \
        return e.code;                                               \
    }                                                                \
    catch (const std::exception& e) {                                \
        cf::set_error(e.what());                                     \
        return CF_RUNTIME;                                           \
    }                                                                \
    return CF_OK;

// Variant that also reports ConvergenceError.best_residual through *stats.
#define CF_API_END_STATS(STATS)                                      \
    }                                                                \
    catch (const cf::CfError& e) {                                   \
        cf::set_error(e.what());                                     \
        if ((STATS) && e.code == CF_CONVERGENCE)                     \
            (STATS)->best_residual = e.best_residual;                \
        return e.code;                                               \
    }                                                                \
    catch (const std::exception& e) {                                \
        cf::set_error(e.what());                                     \
        return CF_RUNTIME;                                           \
    }                                                                \
    return CF_OK;

#ifdef __CUDACC__
#define CF_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t err__ = (call);                                                     \
        if (err__ != cudaSuccess)                                                       \
            throw cf::CfError(CF_RUNTIME, std::string("CUDA error ") +                  \
                                              cudaGetErrorString(err__) + " at " +      \
                                              __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)
#endif
