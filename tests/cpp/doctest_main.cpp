// main() for the reference unit tests under tests/cpp/doctest.h
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
