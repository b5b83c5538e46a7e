// rb_error.h -- thread-local error message shared by the C-ABI translation units.
#pragma once
#include "rcmbfs_b200.h"

#ifdef __cplusplus
extern "C" {
#endif
void rb_set_error(const char* fmt, ...);
#ifdef __cplusplus
}
#endif
