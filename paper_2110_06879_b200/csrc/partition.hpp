// partition.hpp — deterministic bus-graph k-way partition and the per-part
// ownership / boundary-exchange plans of the multi-GPU ADMM.
//
// Ownership: bus i -> part[i]; a generator follows its bus; a branch is solved
// by the owner of its from-bus; a coupling row is owned by the bus that
// consumes it in the bus update (gen rows -> gen's bus, branch rows
// pij,qij,wi,thi -> from-bus, pji,qji,wj,thj -> to-bus).  Per inner iteration
// the only exchanges are, for every cut branch (from and to buses in
// different parts): after the branch phase the solver part sends the four
// to-side x rows to the to-bus part; after the bus/z/y phase the to-bus part
// returns (xbar, z, y) of those rows.  Residual norms are max-reduced (order
// free), all sums stay local in the reference's order, so any partition gives
// results bit-identical to one part.
#ifndef GA_PARTITION_HPP
#define GA_PARTITION_HPP

#include <vector>

#include "network.hpp"

namespace ga {

struct PartPlan {
    int part = 0, parts = 1;
    std::vector<int> gens, buses, rows;  // owned (ascending)
    std::vector<int> lim, unl;           // owned branches by class (ascending)
    // peer q: rows whose x this part sends after the branch phase (= rows
    // whose xbar,z,y it receives after z/y), and rows whose x it receives
    // (= rows whose xbar,z,y it returns).  Branch-major, k = 2,3,6,7.
    std::vector<std::vector<int>> send_x, recv_x;
};

// part[i] for every bus: BFS order from bus 0 over the branch graph (ties by
// index), cut into k contiguous chunks balancing owned branch work (class
// weights, or net.branch_weight when set).  Parts
// may be empty when k exceeds what the graph can fill.
std::vector<int> partition_buses(const Network& net, int k);

// Plan of part p of k (send_x / recv_x sized k, whatever parts are empty).
PartPlan make_plan(const Network& net, const std::vector<int>& part, int p, int k);

}  // namespace ga

#endif
