// tc_dispatch.cu — library-wide launch accounting (gsa_launch_count).
#include "tc.h"

#include <atomic>

namespace gsa_sm100 {

std::atomic<unsigned long long> g_launch_total{0};
void note_launch(int n) { g_launch_total += (unsigned long long)n; }


}  // namespace gsa_sm100
