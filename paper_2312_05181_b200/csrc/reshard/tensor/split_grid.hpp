// reshard/tensor/split_grid.hpp — the reference include path, forwarded: a reference translation unit compiles
// unchanged against this library with -I paper_2312_05181_b200/csrc.  Declares what
// proj/include/reshard/tensor/split_grid.hpp (SplitGrid, grid_refine) declares.
#pragma once

#include "reshard/core.hpp"
