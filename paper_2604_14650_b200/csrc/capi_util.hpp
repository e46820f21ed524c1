// Exception -> status translation for the extern "C" boundary.
#pragma once

#include <exception>
#include <new>
#include <string>

#include "lpm6/common.hpp"

namespace lpm6::capi {

void set_error(const std::string& msg);
void clear_error();

inline int status_of(Errc c) { return static_cast<int>(c) + 1; }

template <class F>
int guard(F&& f) noexcept {
  try {
    clear_error();
    f();
    return 0;
  } catch (const Error& e) {
    set_error(e.what());
    return status_of(e.code());
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return status_of(Errc::InvalidArgument);
  } catch (const std::exception& e) {
    set_error(e.what());
    return status_of(Errc::InvalidArgument);
  } catch (...) {
    set_error("unknown error");
    return status_of(Errc::InvalidArgument);
  }
}

}  // namespace lpm6::capi
