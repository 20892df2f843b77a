// ImageNet-class replica executor (ResNet-50 family) behind the
// ModelExecutor seam (reference proj/include/credo/model.hpp:41-51).
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
  // std::invalid_argument on malformed bytes.
  static std::unique_ptr<CnnModel> from_file(const uint8_t* file, uint64_t len);
  virtual void upload(cudaStream_t st) = 0;
  virtual void reserve(uint32_t max_batch) = 0;
  // d_in: B × input_dim f64 (CHW per image); logits: B × output_dim f32.
  virtual void forward(const double* d_in, uint32_t B, float* logits,
                       cudaStream_t st) = 0;
  virtual uint64_t input_dim() const = 0;
  virtual uint64_t output_dim() const = 0;
  virtual bool softmax() const = 0;
};

}  // namespace cg
