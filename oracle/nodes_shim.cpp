// nodes_shim.cpp -- TEST INFRASTRUCTURE (oracle/).  Error hook for the node
// generator when it is linked into oracle/libnodes_orc.so, the reference
// arm's own copy of the advancing-front generator (geometry.py:105-198):
// bench.py --impl reference must not map the product library, so the node
// set of its workload comes from this separately built object.  The node set
// is pinned to the reference's own outputs (tests/golden/nodes.json), and the
// reference arm re-checks the C2 digest before timing.
#include <string>

namespace {
thread_local std::string g_msg;
}

namespace rbf_detail {
int fail_c(int code, const char* msg) {
  g_msg = msg ? msg : "";
  return code;
}
}  // namespace rbf_detail

extern "C" const char* orc_nodes_last_error(void) { return g_msg.c_str(); }
