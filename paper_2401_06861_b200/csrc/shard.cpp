// Multi-GPU layer (placeholder until the sharded executor lands).
#include "state.hpp"

namespace nqe {

void shard_free(State& s) { (void)s; }
void shard_reset(State& s) { (void)s; }
void shard_flush(State& s) { (void)s; throw NqError{NQ_ERR_INTERNAL, "sharded execution not available"}; }
double shard_norm_sq(State& s) { (void)s; throw NqError{NQ_ERR_INTERNAL, "sharded execution not available"}; }
void shard_expectation(State& s, const uint64_t*, const uint64_t*, const int32_t*, const double*, int, double*) {
    (void)s;
    throw NqError{NQ_ERR_INTERNAL, "sharded execution not available"};
}
void shard_sample(State& s, const double*, uint64_t, uint64_t*, uint64_t*, uint64_t*) {
    (void)s;
    throw NqError{NQ_ERR_INTERNAL, "sharded execution not available"};
}
void shard_get_amplitudes(State& s, uint64_t, uint64_t, double*) {
    (void)s;
    throw NqError{NQ_ERR_INTERNAL, "sharded execution not available"};
}

}  // namespace nqe

extern "C" {

nq_status nq_comm_unique_id(unsigned char out[128]) {
    (void)out;
    return nqe::guard([&] { throw nqe::NqError{NQ_ERR_INTERNAL, "sharded execution not available"}; });
}

nq_status nq_sv_create_sharded(int, int, int, const unsigned char*, const nq_opts*, nq_sv**) {
    return nqe::guard([&] { throw nqe::NqError{NQ_ERR_INTERNAL, "sharded execution not available"}; });
}

nq_status nq_sv_comm_stats(const nq_sv*, int64_t* exchanges, int64_t* bytes_sent) {
    if (exchanges) *exchanges = 0;
    if (bytes_sent) *bytes_sent = 0;
    return NQ_OK;
}
}
