// TEST INFRASTRUCTURE ONLY: main() of the Catch2 stand-in. Every TEST_CASE runs once
// per leaf SECTION (pass k enters the k-th section it meets), like Catch2.
#include "catch2/catch_amalgamated.hpp"

#include <exception>

int main() {
    auto& st = catch_shim::state();
    int cases = 0;
    for (const auto& tc : catch_shim::registry()) {
        ++cases;
        st.test = tc.name;
        for (int pass = 0;; ++pass) {
            st.target = pass;
            st.seen = 0;
            try {
                tc.fn();
            } catch (const catch_shim::RequireFailed&) {
            } catch (const std::exception& e) {
                ++st.failures;
                std::printf("FAILED [%s]: unexpected exception: %s\n", tc.name, e.what());
            }
            if (pass + 1 >= st.seen) break;  // no further section left to enter
        }
    }
    std::printf("%d test cases, %d assertions, %d failed\n", cases, st.assertions, st.failures);
    return st.failures == 0 ? 0 : 1;
}
