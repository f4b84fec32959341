// hanf_graph_internal.h -- the opaque hanf_graph of include/hanf.h: a host
// CSR (graph.hpp:23-69 layout).  Shared by the host builders
// (hanf_host.cpp) and the device builders (hanf_graphgen.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

struct hanf_graph {
  uint64_t n = 0;
  std::vector<uint64_t> offsets{0};
  std::vector<uint32_t> succ;
};

namespace hanf_host_detail {  // defined in hanf_engine.cu (one error slot)
void set_error(const std::string& s);
}
