// api_min.cpp -- temporary: error plumbing only (replaced by api.cpp)
#include "common.h"
namespace pooch {
std::string& tls_error() {
  static thread_local std::string e;
  return e;
}
}  // namespace pooch
extern "C" const char* pooch_last_error(const pooch_ctx*) { return pooch::tls_error().c_str(); }
