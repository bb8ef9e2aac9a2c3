// TEST INFRASTRUCTURE ONLY: runner for the reference's own doctest suites
// (proj/tests/test_*.cpp) built against oracle/doctest_stub/doctest.h.
#define DOCTEST_STUB_IMPLEMENT
#include "doctest.h"
