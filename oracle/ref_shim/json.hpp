// ORACLE — TEST INFRASTRUCTURE ONLY. The reference vendors nlohmann/json as
// vendor/json.hpp (proj/README.md:30-31, gitignored and absent); the same
// library (3.11.3) ships in the image, found by oracle/Makefile.
#pragma once
#include <nlohmann/json.hpp>
