// reshard/util/hash.hpp — the reference include path, forwarded: a reference translation unit compiles
// unchanged against this library with -I paper_2312_05181_b200/csrc.  Declares what
// proj/include/reshard/util/hash.hpp (Fnv1a64, fnv1a64, SplitMix64, splitmix64_next) declares.
#pragma once

#include "reshard/core.hpp"
