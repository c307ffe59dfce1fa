// fetch_stub.cpp -- TEST INFRASTRUCTURE ONLY.  The reference's src/bench.cpp
// (compiled into oracle/_ref for its time_kernel / MTX pipeline) references
// mps::fetch_matrix (include/mps/fetch.hpp:63), whose implementation needs the
// absent cpp-httplib; the suite runner that calls it is never used here.
#include <stdexcept>

#include "mps/fetch.hpp"

namespace mps {
std::filesystem::path fetch_matrix(const std::string& name, const FetchOptions&) {
  throw std::runtime_error("fetch_matrix(" + name + "): no network in this build");
}
}  // namespace mps
