// rb_abi.cu -- error plumbing of the C ABI (include/rcmbfs_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include "rb_error.h"

static thread_local char g_err[1024] = "";

extern "C" void rb_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* rb_last_error(void) { return g_err; }

extern "C" int rb_version(void) { return 1; }
