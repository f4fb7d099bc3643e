// main() for reference unit tests built against the doctest stand-in
// (TEST INFRASTRUCTURE ONLY).
#define DOCTEST_STUB_MAIN
#include "doctest.h"
