// error.h — status/error plumbing for the C ABI (thread-local last error).
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/rn.h"

namespace rn {

rn_status set_error(rn_status s, const std::string &msg);
void count_launch();
void add_launches(int64_t n);
void set_capturing(bool c);
int64_t launch_count();

// Internal exception carrying an rn_status; converted at the ABI boundary.
struct Error : std::runtime_error {
  rn_status status;
  Error(rn_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char *what, const char *file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
    throw Error(RN_ERR_CUDA, buf);
  }
}

}  // namespace rn

#define CUDA_CHECK(x) ::rn::cuda_check((x), #x, __FILE__, __LINE__)
#define LAUNCH_CHECK() (::rn::count_launch(), ::rn::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__))
