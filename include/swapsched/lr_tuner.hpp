// Forwarding header: the reference splits its API per module; this build
// declares everything in swapsched/api.hpp.
#pragma once
#include "swapsched/api.hpp"
