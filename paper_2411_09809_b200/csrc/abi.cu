// Error state, versioning and launch accounting of the glare_b200 C ABI.
#include "common.cuh"

namespace glr {

std::string &last_error() {
  static thread_local std::string msg;
  return msg;
}

void set_error(const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
}

static thread_local uint64_t g_launches = 0;
void count_launch(uint64_t n) { g_launches += n; }

}  // namespace glr

extern "C" {

int glr_version(void) { return (1 << 16) | 0; }

const char *glr_last_error(void) { return glr::last_error().c_str(); }

uint64_t glr_take_launch_count(void) {
  uint64_t n = glr::g_launches;
  glr::g_launches = 0;
  return n;
}

}  // extern "C"
