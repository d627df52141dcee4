// reshard/error.hpp — the reference include path, forwarded: a reference translation unit compiles
// unchanged against this library with -I paper_2312_05181_b200/csrc.  Declares what
// proj/include/reshard/error.hpp (Errc, errc_name, Error, raise) declares.
#pragma once

#include "reshard/core.hpp"
