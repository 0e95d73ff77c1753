// Shim: the reference header annkit/knn_graph.hpp resolves to the B200 framework's C++ API.
#pragma once
#include "annkit_b200.hpp"
