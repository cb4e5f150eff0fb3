// Prompt split (prompt.cpp:14-38) and the /score response body
// (service.cpp:380-391); see prompt.cpp.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

namespace srh {

struct PromptParts {  // prompt.hpp:17-20
  std::vector<int32_t> prefix_tokens;  // system instructions + query context
  std::vector<int32_t> item_tokens;    // document + fixed suffix
};

PromptParts build_prompt(std::string_view system, std::string_view query_context,
                         std::string_view document, int max_seq);

void json_number(std::string& out, double v);
void json_string(std::string& out, std::string_view s);

// score_result_to_json over a flattened result: scores [n_items x n_tasks],
// task_names[t] names column t (any order; emitted sorted by name).
std::string score_result_json(std::string_view request_id, int n_items,
                              const char* const* item_ids, int n_tasks,
                              const char* const* task_names, const double* scores,
                              double attention_units, double linear_units);

}  // namespace srh
