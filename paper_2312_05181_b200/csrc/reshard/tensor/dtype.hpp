// reshard/tensor/dtype.hpp — the reference include path, forwarded: a reference translation unit compiles
// unchanged against this library with -I paper_2312_05181_b200/csrc.  Declares what
// proj/include/reshard/tensor/dtype.hpp (Dtype, dtype_width, dtype_name, dtype_from_name, dtype_from_code) declares.
#pragma once

#include "reshard/core.hpp"
