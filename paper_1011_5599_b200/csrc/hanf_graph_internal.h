// hanf_graph_internal.h -- the opaque hanf_graph of include/hanf.h: a host
// CSR (graph.hpp:23-69 layout).  Shared by the host builders
// (hanf_host.cpp) and the device builders (hanf_graphgen.cu).
#pragma once

#include <cstdint>
#include <memory>
#include <new>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

// resize() without zero-filling: every builder writes all the elements it
// sizes, and zero-filling the 17 GB of a config-5 graph first cost seconds
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible_v<U>) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};

struct hanf_graph {
  uint64_t n = 0;
  std::vector<uint64_t, DefaultInitAlloc<uint64_t>> offsets{0};
  std::vector<uint32_t, DefaultInitAlloc<uint32_t>> succ;
};

namespace hanf_host_detail {  // defined in hanf_engine.cu (one error slot)
void set_error(const std::string& s);
}
