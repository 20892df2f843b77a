// Shared helpers for the credo B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>

namespace cg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define CG_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      throw ::cg::CudaError(std::string(#call) + ": " +                      \
                            cudaGetErrorString(e_) + " @" + __FILE__ + ":" + \
                            std::to_string(__LINE__));                       \
  } while (0)

// Every kernel launch site goes through CG_CHECK_LAUNCH, which also counts
// the launch (reported as gpu_launches by bench.py).
uint64_t launch_counter_add(uint64_t n);
#define CG_CHECK_LAUNCH()              \
  do {                                 \
    CG_CUDA(cudaGetLastError());       \
    ::cg::launch_counter_add(1);       \
  } while (0)

// Optional per-kernel-class device timing (CUDA events on the launching
// stream), used by bench.py to attribute step time to the dominant kernel.
enum TimerClass : int {
  kTimeGemm = 0,   // conv_gemm launches
  kTimeChain = 1,  // SHA-256 chain jobs
  kTimeAgree = 2,  // softmax/top-k, select_quorum, manifest, Merkle trees
  kTimeAux = 3,    // CNN input prep, gathers, pools
  kTimeComm = 4,   // NCCL exchange (replica-parallel groups)
  kTimeClasses = 5
};
void timer_begin(cudaStream_t st, int cls);
void timer_end(cudaStream_t st, int cls);

constexpr int kNumSMs = 148;

// Runs f() once per device: cudaFuncSetAttribute opt-ins (dynamic shared
// memory above 48 KB) apply to the current device only, so a process that
// drives several GPUs must set them on each.
template <typename F>
void once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int d = 0;
  CG_CUDA(cudaGetDevice(&d));
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) {
  return (a + b - 1) / b;
}

}  // namespace cg
