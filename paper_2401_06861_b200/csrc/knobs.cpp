#include "knobs.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

extern char** environ;

namespace nqe {

int env_option(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return (e && *e) ? std::atoi(e) : dflt;
}

std::string env_option_str(const char* name) {
    const char* e = std::getenv(name);
    return e ? std::string(e) : std::string();
}

int ab_knob(const char* name, int dflt) {
#ifdef NQ_AB_KNOBS
    return env_option(name, dflt);
#else
    (void)name;
    return dflt;
#endif
}

std::string plan_env_fingerprint() {
    static const char* const diag[] = {"NQ_PLAN_TRACE", "NQ_SHARD_TRACE", "NQ_SHARD_TIMING", "NQ_JIT_DUMP",
                                       "NQ_BATCH_TIMING", "NQ_SEGV_TRACE", "NQ_NCCL_LIB"};
    std::vector<std::string> kv;
    for (char** e = environ; e && *e; ++e) {
        if (std::strncmp(*e, "NQ_", 3) != 0) continue;
        const char* eq = std::strchr(*e, '=');
        const std::string name(*e, eq ? size_t(eq - *e) : std::strlen(*e));
        if (std::any_of(std::begin(diag), std::end(diag), [&](const char* d) { return name == d; })) continue;
#ifndef NQ_AB_KNOBS
        // A/B switches are ignored by this build, so they cannot diverge
        static const char* const honoured[] = {"NQ_JIT", "NQ_JIT_PX", "NQ_TILE_SV", "NQ_TILE_DM", "NQ_EXCHANGE",
                                               "NQ_FUSED_EXCHANGE", "NQ_COMM"};
        if (std::none_of(std::begin(honoured), std::end(honoured), [&](const char* d) { return name == d; }))
            continue;
#endif
        kv.emplace_back(*e);
    }
    std::sort(kv.begin(), kv.end());
    std::string out;
    for (const auto& s : kv) out += s + ";";
    return out;
}

}  // namespace nqe
