// SPDX-License-Identifier: Apache-2.0
// Runner for the reference's own Catch2 suites compiled unmodified against include/chunktrain
// (see tests/test_cpp_reference_suites.py).
#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
