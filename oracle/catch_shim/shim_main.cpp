#define CATCH_SHIM_MAIN
#include <catch2/catch_amalgamated.hpp>
