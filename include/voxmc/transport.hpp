// transport.hpp — reference-compatible include path; the B200 API lives in voxmc.hpp.
#pragma once
#include "voxmc/voxmc.hpp"
