// C5 from C++ through the drop-in library: fastnn::reciprocal_match_sharded
// over a native NCCL communicator must return exactly what
// fastnn::reciprocal_match returns on the same maps (MatchSet in order, and
// the RunReport except its four timing fields).
//
//   c5_sharded H W backend metric           one rank (the GPU box has one GPU)
//   FNL_RANK=r FNL_NRANKS=n FNL_ID_FILE=p c5_sharded ...   one process per GPU;
//       rank 0 writes the NCCL id to p, the others read it
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>

#include "fastnn/io.hpp"
#include "fastnn/reciprocal.hpp"
#include "fastnn/sharded.hpp"

namespace fastnn::b200 {
void set_device(int device);
}

int main(int argc, char** argv) {
    using namespace fastnn;
    const std::uint32_t H = argc > 1 ? std::atoi(argv[1]) : 192, W = argc > 2 ? std::atoi(argv[2]) : 144;
    const std::string backend = argc > 3 ? argv[3] : "single", metric = argc > 4 ? argv[4] : "dot";
    const int rank = std::getenv("FNL_RANK") ? std::atoi(std::getenv("FNL_RANK")) : 0;
    const int nranks = std::getenv("FNL_NRANKS") ? std::atoi(std::getenv("FNL_NRANKS")) : 1;
    const char* id_file = std::getenv("FNL_ID_FILE");
    if (nranks > 1) b200::set_device(rank);

    NcclCommunicator::Id id{};
    if (rank == 0) {
        id = NcclCommunicator::unique_id();
        if (nranks > 1) {
            std::ofstream(std::string(id_file) + ".tmp", std::ios::binary).write((const char*)id.data(), 128);
            std::rename((std::string(id_file) + ".tmp").c_str(), id_file);
        }
    } else {
        for (;;) {
            std::ifstream f(id_file, std::ios::binary);
            if (f && f.read((char*)id.data(), 128)) break;
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    NcclCommunicator comm(id, nranks, rank);

    const FeatureMap D1 = gen_random(H, W, 24, 2606, true);
    const FeatureMap D2 = gen_random(H, W, 24, 2607, true);
    MatchConfig cfg;
    cfg.grid_stride = 8;
    cfg.metric = metric_from_string(metric);
    const NnBackend be = backend_from_string(backend);
    const MatchOutcome sharded = reciprocal_match_sharded(D1, D2, cfg, be, comm);
    const MatchOutcome whole = reciprocal_match(D1, D2, cfg, be);
    RunReport a = sharded.report, b = whole.report;
    a.subsample_us = b.subsample_us = a.forward_nn_us = b.forward_nn_us = 0;
    a.reverse_nn_us = b.reverse_nn_us = a.harvest_us = b.harvest_us = 0;
    const bool same = sharded.matches.pairs == whole.matches.pairs && a == b;
    std::cout << "rank " << rank << "/" << nranks << " " << backend << " " << metric << " matches "
              << sharded.matches.pairs.size() << " vs " << whole.matches.pairs.size()
              << (same ? " IDENTICAL" : " DIFFER") << std::endl;
    return same ? 0 : 1;
}
