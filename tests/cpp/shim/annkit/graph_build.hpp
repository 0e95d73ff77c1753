// Shim: the reference header annkit/graph_build.hpp resolves to the B200 framework's C++ API.
#pragma once
#include "annkit_b200.hpp"
