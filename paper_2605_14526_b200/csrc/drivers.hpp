// Host drivers over the public C ABI (drivers.cpp): system identification and
// the finite-difference gradient check.  Linked into both the product and the
// oracle library, each wrapping them as hd_run_identify(_file) /
// hd_run_gradcheck.
#pragma once
#include <string>

struct hd_scene;

namespace heterodyn_driver {
// Returns an hd_status; on failure *error holds the message.
int run_identify(const std::string& problem_text, const std::string& out_dir, std::string* result, bool* stalled,
                 std::string* error);
int run_identify_file(const std::string& path, const std::string& out_dir, std::string* result, bool* stalled,
                      std::string* error);
int run_gradcheck(const hd_scene* scene, const char* vars_csv, const char* out_path, std::string* report,
                  bool* pass, std::string* error);
int run_simulate(const hd_scene* scene, const char* out_dir, std::string* summary, std::string* error);
}  // namespace heterodyn_driver
