// Self-test of tests/cpp/refshim/doctest.h: SUBCASE re-runs the test case so
// every leaf path runs exactly once, like doctest (checked against the known
// leaf sequence of a nested case).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <string>
#include <vector>

static std::vector<std::string> g_trace;

TEST_CASE("nested subcases") {
  std::string path = "T";
  SUBCASE("A") {
    path += "A";
    SUBCASE("A1") { path += "1"; }
    SUBCASE("A2") { path += "2"; }
  }
  SUBCASE("B") { path += "B"; }
  g_trace.push_back(path);
}

TEST_CASE("trace is doctest's leaf order") {
  CHECK(g_trace == std::vector<std::string>{"TA1", "TA2", "TB"});
  CHECK(0.1 + 0.2 == doctest::Approx(0.3));
  CHECK_FALSE(1.0 == doctest::Approx(1.001));
  CHECK(1.0 == doctest::Approx(1.001).epsilon(0.01));
  CHECK_THROWS_AS(throw std::runtime_error("x"), std::runtime_error);
}
