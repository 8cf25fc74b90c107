// Host side of the GPU dataset loader: the header line and the MESSAGE of the
// first failing record. The data path is the device (ingest.cu); this file
// only turns "line k fails" into the reference's exact text, by running the
// reference's checks (dataset.cpp:73-168) on that single line with the same
// JSON library (nlohmann/json 3.11, a dependency of the reference build).
#include <json.hpp>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "ingest_host.hpp"

namespace pars_b200 {

namespace {

using json = nlohmann::json;

std::string positive_int_error(const json& v, const char* field) {
  if (!v.is_number_integer() || v.get<int64_t>() < 1)
    return std::string("field '") + field + "' must be a positive integer";
  return "";
}

int64_t median_floor(std::vector<int64_t> s) {
  std::sort(s.begin(), s.end());
  const size_t n = s.size();
  if (n % 2 == 1) return s[n / 2];
  return (s[n / 2 - 1] + s[n / 2]) / 2;
}

int64_t token_count(const std::string& text) {
  int64_t count = 0;
  bool in_token = false;
  for (unsigned char c : text) {
    if (c == ' ' || (c >= 9 && c <= 13)) {
      in_token = false;
    } else if (!in_token) {
      in_token = true;
      ++count;
    }
  }
  return count;
}

}  // namespace

std::string ingest_header_error(const std::string& line, int64_t* embedding_dim) {
  try {
    json header = json::parse(line);
    if (header.value("format", "") != "pars.dataset") return "not a pars dataset (bad format field)";
    if (header.value("version", 0) != 1)
      return "unsupported version " + std::to_string(header.value("version", 0));
    *embedding_dim = header.value("embedding_dim", int64_t{0});
    if (*embedding_dim < 0) return "embedding_dim must be >= 0";
  } catch (const json::exception& e) {
    return std::string("malformed header: ") + e.what();
  }
  return "";
}

std::string ingest_record_error(const std::string& line, bool duplicate, int64_t embedding_dim,
                                bool* has_embedding) {
  *has_embedding = false;
  json j;
  try {
    j = json::parse(line);
  } catch (const json::exception& e) {
    return std::string("malformed record: ") + e.what();
  }
  if (!j.is_object()) return "record must be an object";
  if (!j.contains("id") || !j["id"].is_string() || j["id"].get<std::string>().empty())
    return "missing or invalid field 'id'";
  if (duplicate) return "duplicate id '" + j["id"].get<std::string>() + "'";
  if (!j.contains("prompt") || !j["prompt"].is_string()) return "missing or invalid field 'prompt'";
  std::vector<int64_t> samples;
  if (j.contains("output_len_samples")) {
    const json& arr = j["output_len_samples"];
    if (!arr.is_array() || arr.empty()) return "'output_len_samples' must be a non-empty array";
    for (const json& v : arr) {
      const std::string e = positive_int_error(v, "output_len_samples");
      if (!e.empty()) return e;
      samples.push_back(v.get<int64_t>());
    }
  }
  if (j.contains("output_len")) {
    const std::string e = positive_int_error(j["output_len"], "output_len");
    if (!e.empty()) return e;
    if (!samples.empty() && j["output_len"].get<int64_t>() != median_floor(samples))
      return "output_len does not equal the median of output_len_samples";
  } else if (samples.empty()) {
    return "missing field 'output_len'";
  }
  if (j.contains("embedding")) {
    const json& arr = j["embedding"];
    if (!arr.is_array()) return "'embedding' must be an array";
    for (const json& v : arr)
      if (!v.is_number()) return "'embedding' entries must be numbers";
    if (static_cast<int64_t>(arr.size()) != embedding_dim) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "embedding length %zu does not match declared dimension %lld",
                    arr.size(), static_cast<long long>(embedding_dim));
      return buf;
    }
    *has_embedding = true;
  }
  if (j.contains("prompt_len")) {
    const std::string e = positive_int_error(j["prompt_len"], "prompt_len");
    if (!e.empty()) return e;
  } else if (token_count(j["prompt"].get<std::string>()) < 1) {
    return "prompt has no tokens and no prompt_len";
  }
  return "";
}

std::vector<int64_t> ingest_parse_samples(const std::string& arr) {
  std::vector<int64_t> out;
  for (const json& v : json::parse(arr)) out.push_back(v.get<int64_t>());
  return out;
}

}  // namespace pars_b200
