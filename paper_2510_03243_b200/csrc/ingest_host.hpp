// Host error path of the GPU dataset loader (ingest_host.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace pars_b200 {

// "" when the header line is valid (sets *embedding_dim), else the
// reference's message without the "path: line 1: " prefix.
std::string ingest_header_error(const std::string& line, int64_t* embedding_dim);

// The reference's checks on one record line (dataset.cpp:103-168); "" when it
// passes (then *has_embedding says whether it carries an embedding array).
std::string ingest_record_error(const std::string& line, bool duplicate, int64_t embedding_dim,
                                bool* has_embedding);

// The integers of a validated output_len_samples array.
std::vector<int64_t> ingest_parse_samples(const std::string& arr);

}  // namespace pars_b200
