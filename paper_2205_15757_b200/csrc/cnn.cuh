// ImageNet-class replica executors (ResNet-50/101/152 bottleneck v1.5,
// VGG-16, MobileNetV2)
// behind the ModelExecutor seam (reference proj/include/credo/model.hpp:
// 41-51). The reference has no CNN path (its SPEC.md:8 replaces it with
// LinearToyModel); the CPU restatement used as parity oracle is torchvision's
// fp32 forward of the same state dict.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

namespace cg {

class CnnModel {
 public:
  virtual ~CnnModel() = default;
  // Parses the canonical CNN model file. Throws
  // std::invalid_argument on malformed bytes or an unsupported arch.
  static std::unique_ptr<CnnModel> from_file(const uint8_t* file, uint64_t len);
  virtual void upload(cudaStream_t st) = 0;
  virtual void reserve(uint32_t max_batch) = 0;
  // Replica-independent input stage (f64 CHW -> bf16 conv1 operand); the
  // group runs it once per batch and shares it across replicas.
  virtual void prepare_input(const double* d_in, uint32_t B, void* prepped,
                             cudaStream_t st) = 0;
  virtual size_t prepared_bytes(uint32_t B) const = 0;
  // Models with equal prep_kind() can share one prepared input.
  virtual std::string prep_kind() const = 0;
  // logits: B × output_dim f32. prepped == nullptr -> prepares internally.
  virtual void forward(const double* d_in, uint32_t B, float* logits,
                       cudaStream_t st, const void* prepped = nullptr) = 0;
  virtual uint64_t input_dim() const = 0;
  virtual uint64_t output_dim() const = 0;
  virtual bool softmax() const = 0;
  virtual std::string arch() const = 0;
  virtual double flops_per_image() const = 0;  // 2 × MACs of the forward
};

// The forward of several replicas of one architecture executed layer by
// layer with one grouped GEMM launch per layer (3x the tiles of a single
// replica: small late-stage layers fill the GPU in balanced waves).
class CnnGroupPlan {
 public:
  virtual ~CnnGroupPlan() = default;
  // nullptr when the models cannot be grouped (different architectures or
  // input shapes). prepped: the shared conv1 operand; logits[r]: B x classes.
  static std::unique_ptr<CnnGroupPlan> build(const std::vector<CnnModel*>& models, uint32_t B,
                                             const void* prepped,
                                             const std::vector<float*>& logits);
  virtual void run(cudaStream_t st) = 0;
  virtual uint32_t batch() const = 0;
};

}  // namespace cg
