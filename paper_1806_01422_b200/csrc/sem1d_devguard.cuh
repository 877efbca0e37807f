// sem1d_devguard.cuh -- per-device launch caches and the plan device guard (host only).
#pragma once

#include <cuda_runtime.h>

namespace sem1d {

// Launch caches are per device: cudaFuncSetAttribute and the occupancy query are
// properties of a (kernel, device) pair, so a process that drives several GPUs keeps one
// entry per device ordinal.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
struct DevCache {
  int v[kMaxDevices] = {};
  int& here() { return v[current_device()]; }
};
inline int device_sms() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
  return sms > 0 ? sms : 148;
}

// Makes a plan's device current for the duration of a C-ABI call (restored on exit), so a
// plan created on device d launches there whatever device the caller has current.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace sem1d
