// fs_internal.h — helpers shared by the translation units of the library.
#pragma once
#include <string>

namespace fs {
extern thread_local std::string g_last_error;
int set_error(int code, const char* fmt, ...);
}  // namespace fs
