// TEST INFRASTRUCTURE ONLY: entry point for the doctest shim.
#define DOCTEST_SHIM_MAIN
#include "doctest.h"
