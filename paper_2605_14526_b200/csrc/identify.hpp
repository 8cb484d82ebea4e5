// System-identification driver over the public C ABI (identify.cpp); linked
// into both the product and the oracle library, each wrapping it as
// hd_run_identify / hd_run_identify_file.
#pragma once
#include <string>

namespace heterodyn_driver {
// Returns an hd_status; on failure *error holds the message.
int run_identify(const std::string& problem_text, const std::string& out_dir, std::string* result, bool* stalled,
                 std::string* error);
int run_identify_file(const std::string& path, const std::string& out_dir, std::string* result, bool* stalled,
                      std::string* error);
}  // namespace heterodyn_driver
