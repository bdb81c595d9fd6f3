// host_common.hpp -- error plumbing for the C ABI: C++ exceptions inside,
// status codes + thread-local messages at the boundary (include/atkg.h).
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/atkg.h"

namespace atkg {

struct Inval : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NanInput : std::invalid_argument { NanInput() : std::invalid_argument("input contains NaN") {} };
struct Infeasible : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct Unsupported : std::runtime_error { using std::runtime_error::runtime_error; };

[[noreturn]] inline void throw_inval(const char* m) { throw Inval(m); }

void set_last_error(const std::string& m);

// re-raises a status code returned by another entry point (inside guarded())
inline void rethrow(int rc) {
  if (rc == ATKG_OK) return;
  const std::string m = atkg_last_error();
  switch (rc) {
    case ATKG_ENAN: throw NanInput();
    case ATKG_EINFEASIBLE: throw Infeasible(m);
    case ATKG_ECUDA: throw CudaError(m);
    case ATKG_EUNSUPPORTED: throw Unsupported(m);
    default: throw Inval(m);
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ATKG_OK;
  } catch (const NanInput& e) {
    set_last_error(e.what());
    return ATKG_ENAN;
  } catch (const Inval& e) {
    set_last_error(e.what());
    return ATKG_EINVAL;
  } catch (const Infeasible& e) {
    set_last_error(e.what());
    return ATKG_EINFEASIBLE;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return ATKG_ECUDA;
  } catch (const Unsupported& e) {
    set_last_error(e.what());
    return ATKG_EUNSUPPORTED;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ATKG_EINVAL;
  }
}

}  // namespace atkg
