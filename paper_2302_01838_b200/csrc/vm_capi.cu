// C-ABI plumbing: error strings, version, layout query, FFMA peak probe.
#include "vm_common.cuh"

#include <string>

namespace vm {
static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_check(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return VM_ERR_CUDA;
}

// Dependent-chain-free FFMA stream: 8 independent accumulators per thread.
__global__ void ffma_probe_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}
}  // namespace vm

extern "C" const char* vm_last_error(void) { return vm::g_last_error.c_str(); }

extern "C" const char* vm_version(void) { return "vmap_b200 0.1 sm_100a"; }

extern "C" int vm_model_layout(const VmArch* arch, VmLayout* out) {
  if (!arch || !out) return VM_ERR_SHAPE;
  int rc = vm::compute_layout(*arch, *out);
  if (rc) vm::set_error("vm_model_layout: unsupported architecture");
  return rc;
}

extern "C" int vm_ffma_peak(int iters, float* tflops, void* stream) {
  cudaStream_t s = cudaStream_t(stream);
  int dev = 0, sms = 0;
  VM_CUDA(cudaGetDevice(&dev));
  VM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* out = nullptr;
  VM_CUDA(cudaMallocAsync(&out, 4, s));
  cudaEvent_t e0, e1;
  VM_CUDA(cudaEventCreate(&e0));
  VM_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  vm::ffma_probe_kernel<<<blocks, threads, 0, s>>>(out, 64, 0.999f, 0.001f);  // warm-up
  VM_CUDA(cudaEventRecord(e0, s));
  vm::ffma_probe_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
  VM_CUDA(cudaEventRecord(e1, s));
  VM_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  VM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *tflops = float(2.0 * 8.0 * double(iters) * blocks * threads / (ms * 1e-3) / 1e12);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  VM_CUDA(cudaFreeAsync(out, s));
  return VM_OK;
}
