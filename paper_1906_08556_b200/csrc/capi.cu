// Library-level C ABI: version and thread-local error reporting.
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace tvk {
static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace tvk

extern "C" int tvk_version(void) { return 100; }

extern "C" int tvk_last_error(char* buf, int64_t n) {
  int len = (int)strlen(tvk::g_err);
  if (buf && n > 0) {
    int64_t k = len < n - 1 ? len : n - 1;
    memcpy(buf, tvk::g_err, (size_t)k);
    buf[k] = 0;
  }
  return len;
}
