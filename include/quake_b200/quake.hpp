// quake_b200/quake.hpp — umbrella for the C++ drop-in of the reference's
// quake:: operator API.
//
// The drop-in mirrors the reference's header layout under
// include/quake_b200/quake/ (bitcore.hpp, buffer.hpp, kernels.hpp,
// nonlin.hpp), so reference code that includes "quake/kernels.hpp" or
// "quake/nonlin.hpp" compiles unchanged with -I <repo>/include/quake_b200
// and links libquake_b200.so; the reference's own tests/test_kernels.cpp,
// test_nonlin.cpp and test_bitcore.cpp are built that way (tests/cpp/Makefile)
// and run on the B200. This header includes all four.
#ifndef QUAKE_B200_QUAKE_HPP_
#define QUAKE_B200_QUAKE_HPP_

#include "quake/bitcore.hpp"
#include "quake/buffer.hpp"
#include "quake/kernels.hpp"
#include "quake/nonlin.hpp"

#endif  // QUAKE_B200_QUAKE_HPP_
