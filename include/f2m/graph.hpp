// Compatibility include: the reference header f2m/graph.hpp maps onto the single B200 API header.
#pragma once
#include "f2m/api.hpp"
