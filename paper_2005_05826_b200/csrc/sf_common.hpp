// Shared helpers for the stripefrac B200 library: thread-local error text.
#pragma once

#include <string>

namespace sf {

// Last error on the calling thread (sf_last_error()).
void set_error(const std::string& msg);
const char* last_error();

}  // namespace sf
