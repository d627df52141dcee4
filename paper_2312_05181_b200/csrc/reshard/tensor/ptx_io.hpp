// reshard/tensor/ptx_io.hpp — the reference include path, forwarded: a reference translation unit compiles
// unchanged against this library with -I paper_2312_05181_b200/csrc.  Declares what
// proj/include/reshard/tensor/ptx_io.hpp (ptx_encode, ptx_decode, ptx_write_file, ptx_read_file, ptx_encoded_size) declares.
#pragma once

#include "reshard/checkpoint.hpp"
