// Drop-in implementation of the reference's predictor/scheduler translation
// units (proj/src/{error,features,scorer,pairs,train,scheduler,metrics}.cpp)
// over the C ABI of include/pars_cuda.h. Compiled against the reference's
// UNMODIFIED public headers (proj/include/pars/*.hpp), so it links into any
// program built against them in place of those .cpp files.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pars/dataset.hpp"
#include "pars/error.hpp"
#include "pars/features.hpp"
#include "pars_cuda.h"

namespace pars::b200 {

// The process-wide device context (device PARS_DEVICE, default 0). Throws
// pars::Error if libpars_cuda has no usable sm_100 device: there is no CPU
// fallback for the hot path.
pars_ctx* ctx();

// Rethrows a C-ABI failure as pars::Error carrying the library's message.
void check(int64_t rc);

pars_extractor to_c(const FeatureExtractor& ex);

// Text arena + offsets for a dataset (or a single record).
struct Packed {
  std::string text;
  std::vector<int64_t> offsets;
};
Packed pack(const Dataset& ds);
Packed pack(const PromptRecord& rec);

// Reference-identical validation of a record against the embedding
// extractor (features.cpp:64-73); returns the dense row.
void check_embedding(const FeatureExtractor& ex, const PromptRecord& rec);

// RAII device CSR.
struct DeviceFeatures {
  pars_features* f = nullptr;
  DeviceFeatures() = default;
  DeviceFeatures(const DeviceFeatures&) = delete;
  DeviceFeatures& operator=(const DeviceFeatures&) = delete;
  ~DeviceFeatures() {
    if (f) pars_features_free(f);
  }
};

// extract_all on the GPU into a device CSR.
void extract_device(const FeatureExtractor& ex, const Dataset& ds, DeviceFeatures& out);
// Upload host FeatureVecs as a device CSR.
void upload(uint32_t dim, const std::vector<const FeatureVec*>& rows, DeviceFeatures& out);
std::vector<FeatureVec> download(const DeviceFeatures& f);

}  // namespace pars::b200
