// Compatibility header: the reference splits these types across proj/include/ooc/*.hpp;
// ooc-b200 keeps them together in ooc/core.hpp.
#pragma once
#include "ooc/core.hpp"
