// Reference header path (proj/include/tzc/workloads.hpp) kept for drop-in C++ callers:
// the B200 backend declares the whole API in tzc/tzc.hpp.
#pragma once
#include "tzc/tzc.hpp"
