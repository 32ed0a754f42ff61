// Thread-local error reporting for the C-ABI (hc_last_error).
#pragma once
#include <cstdarg>
#include <cstdio>

#include "hcinfer.h"

namespace hc {

inline char* last_error_buf() {
  static thread_local char buf[1024] = "";
  return buf;
}

inline hc_status fail(hc_status code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(last_error_buf(), 1024, fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace hc
