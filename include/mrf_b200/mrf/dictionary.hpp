// mrf/dictionary.hpp -- include shim: code written against the reference's
// proj/include/mrf/dictionary.hpp compiles unchanged with -I include/mrf_b200
// (all declarations live in the single drop-in header).
#pragma once
#include "../mrf.hpp"
