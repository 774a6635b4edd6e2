// host_util.h — host-side helpers shared by the C-ABI translation units
// (tvs_api.cu, train.cu): error type and CUDA check macro, the thread-local
// last-error string, the guarded() boundary (no C++ exception crosses the C
// ABI), device guard and TMA descriptor encoding.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/tvs_b200.h"

namespace tvs_host {

std::string& last_error();  // thread-local, defined in tvs_api.cu

struct TvsError : std::runtime_error {
  int code;
  TvsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TVS_CUDA(call)                                                                                     \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      throw tvs_host::TvsError(TVS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ \
                                               ":" + std::to_string(__LINE__) + ")");                       \
  } while (0)

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    TVS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw TvsError(TVS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp16 NHWC activation [B][H][W][C] (C = 64, or 128 = a hi|lo pair row) as a
// 4-D tensor map, SW128, box (64, box_px, 1, 1).  A padded buffer
// [B][H+2*pad][W+2*pad][C] is described by passing its interior origin as
// `base` and pad = 1: the borders are never read (TMA zero-fills outside the
// W x H extent, which is the convolution's zero padding).
inline CUtensorMap make_act_map(void* base, int B, int H, int W, int box_px, int C = 64, int pad = 0) {
  CUtensorMap m;
  const cuuint64_t rb = (cuuint64_t)C * 2;
  const cuuint64_t Wp = (cuuint64_t)W + 2 * pad, Hp = (cuuint64_t)H + 2 * pad;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {rb, Wp * rb, Hp * Wp * rb};
  cuuint32_t box[4] = {64, (cuuint32_t)box_px, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TvsError(TVS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// Restores the caller's current device on scope exit: the ABI may run on any
// thread and must not change that thread's device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) TVS_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TVS_OK;
  } catch (const TvsError& e) {
    last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return TVS_E_CUDA;
  } catch (...) {
    last_error() = "unknown error";
    return TVS_E_CUDA;
  }
}

}  // namespace tvs_host
