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

// ALN1 frame-record walk (read_alignment's decoder, io_formats.py:154-227): host code, no device.
// words = one utterance's u32 stream [count_t, (component, weight bits) * count_t] for t < n_frames.
extern "C" int tvk_aln1_scan(const uint32_t* words, int64_t n_words, int64_t n_frames, int64_t* starts,
                             int64_t* counts, int64_t* end) {
  int64_t pos = 0;
  for (int64_t t = 0; t < n_frames; t++) {
    if (pos >= n_words) {
      tvk::set_error("aln1: frame record shorter than declared (entry count)");
      return TVK_ERR_INVALID;
    }
    const int64_t k = words[pos];
    starts[t] = pos;
    counts[t] = k;
    pos += 1 + 2 * k;
  }
  if (pos > n_words) {
    tvk::set_error("aln1: frame record shorter than declared (frame entries)");
    return TVK_ERR_INVALID;
  }
  *end = pos;
  return TVK_OK;
}
