// unit_main.cpp -- TEST INFRASTRUCTURE ONLY: runner for the Catch2 shim.
// usage: unit_main [substring ...] [!substring ...]   (runs the test cases
// whose name contains any of the plain substrings -- all when none -- and none
// of the !-prefixed ones).  Prints one line per failure and a summary; exit 0
// iff every selected case passed.
#include <cstdio>
#include <cstring>

#include "catch_amalgamated.hpp"

int main(int argc, char** argv) {
    int run = 0, failed = 0;
    for (const auto& c : shim::registry()) {
        bool any_include = false, selected = false, excluded = false;
        for (int i = 1; i < argc; ++i) {
            if (argv[i][0] == '!') {
                excluded |= std::strstr(c.name, argv[i] + 1) != nullptr;
            } else {
                any_include = true;
                selected |= std::strstr(c.name, argv[i]) != nullptr;
            }
        }
        selected = (selected || !any_include) && !excluded;
        if (!selected) continue;
        ++run;
        try {
            c.fn();
        } catch (const shim::Failure& f) {
            ++failed;
            std::printf("FAILED: %s\n  %s\n", c.name, f.what());
        } catch (...) {
            ++failed;
            std::printf("FAILED: %s\n  unexpected exception: %s\n", c.name, shim::describe_current().c_str());
        }
    }
    std::printf("test cases: %d | passed: %d | failed: %d | assertions: %ld\n", run, run - failed, failed,
                shim::assertions());
    return failed ? 1 : 0;
}
