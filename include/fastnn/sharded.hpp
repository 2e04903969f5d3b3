// fastnn/sharded.hpp -- EXTENSION of the B200 build (the reference has no
// distributed code): config C5 from C++, one oversized pair with the target
// columns of every NN pass split over the GPUs of a node and the per-query
// (distance, index) winner keys MIN-all-reduced with NCCL.  Every rank gets
// the MatchOutcome of fastnn::reciprocal_match on the same maps, bit for bit.
#pragma once

#include <array>
#include <cstdint>

#include "fastnn/reciprocal.hpp"

struct fnl_comm;

namespace fastnn {

// One NCCL communicator per process / GPU (the calling thread's device, see
// fastnn::b200::set_device).  Rank 0 creates the id and hands its 128 bytes to
// the other ranks out of band; construction is collective.
class NcclCommunicator {
public:
    using Id = std::array<std::uint8_t, 128>;
    static Id unique_id();
    NcclCommunicator(const Id& id, int nranks, int rank);
    ~NcclCommunicator();
    NcclCommunicator(const NcclCommunicator&) = delete;
    NcclCommunicator& operator=(const NcclCommunicator&) = delete;
    int size() const { return nranks_; }
    int rank() const { return rank_; }
    fnl_comm* handle() const { return comm_; }

private:
    fnl_comm* comm_ = nullptr;
    int nranks_ = 0, rank_ = 0;
};

// reciprocal_match with the target columns sharded over `comm` (every rank
// passes identical D1 / D2 / cfg / backend).
MatchOutcome reciprocal_match_sharded(const FeatureMap& D1, const FeatureMap& D2, const MatchConfig& cfg,
                                      NnBackend backend, const NcclCommunicator& comm);

}  // namespace fastnn
