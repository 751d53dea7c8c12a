// network.hpp — host-side power network model, MATPOWER reader and the
// coupling layout that fixes the device row order.
//
// Semantics follow the reference (proj/src/netdata.{hpp,cpp},
// proj/src/decomp.{hpp,cpp}): identical indexing (file order, status-0
// generators/branches dropped), per-unit conversion, admittances of the
// pi-model with complex tap.  The parse itself is new code (single pass over
// the text, strtod tokens).
#ifndef GA_NETWORK_HPP
#define GA_NETWORK_HPP

#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace ga {

class ParseError : public std::runtime_error {
public:
    explicit ParseError(const std::string& w) : std::runtime_error(w) {}
};

struct Bus {
    int id = 0;
    int type = 1;  // 1 PQ, 2 PV, 3 REF
    double pd = 0, qd = 0, gs = 0, bs = 0, vmin = 0, vmax = 0;
};

struct Gen {
    int bus = 0;
    double pmin = 0, pmax = 0, qmin = 0, qmax = 0;
    double c2 = 0, c1 = 0, c0 = 0;
};

// gii bii gij bij gji bji gjj bjj (netdata.hpp:37-43)
struct Admittance {
    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

struct Line {
    int from = 0, to = 0;
    double r = 0, x = 0, b = 0, tap = 1, shift = 0, rate = 0;
    Admittance y;
    bool limited() const { return rate > 0.0; }
};

struct Network {
    double base_mva = 100.0;
    std::vector<Bus> buses;
    std::vector<Gen> gens;
    std::vector<Line> lines;
    std::unordered_map<int, int> bus_index;
    int ref_bus = -1;
    // optional per-branch work weights for the bus partition (e.g. measured
    // TRON steps, gridadmm_session_branch_costs); empty = class weights
    std::vector<int> branch_weight;

    int nb() const { return static_cast<int>(buses.size()); }
    int ng() const { return static_cast<int>(gens.size()); }
    int nl() const { return static_cast<int>(lines.size()); }
    int m() const { return 2 * ng() + 8 * nl(); }
};

Admittance derive_admittance(double r, double x, double b, double tap, double shift);
// pij, qij, pji, qji at a voltage point (netdata.cpp:33-45), pinned sincos.
void branch_flows_host(const Admittance& y, double vi, double vj, double thi, double thj,
                       double out[4]);

Network parse_matpower(const std::string& text);
Network load_matpower(const std::string& path);

// Bus-owned row CSR in the reference's CouplingLayout order
// (decomp.cpp:7-31): per bus, groups [w | theta | gen_p | gen_q | flow_p |
// flow_q]; grp has 7 offsets per bus.
struct BusCsr {
    std::vector<int> grp;   // 7 * nb
    std::vector<int> rows;  // m
};
BusCsr build_bus_csr(const Network& net);

// Device storage order of the m coupling rows ("bus-major quads"): bus i
// owns one contiguous segment [seg, end) holding its generators' (p, q) row
// pairs in generator order, then — from a 4-aligned qstart — one quad
// (p, q, w, theta) per incident branch end in branch order: the rows
// (pij, qij, wi, thi) of a branch at its from-bus, (pji, qji, wj, thj) at its
// to-bus.  Each reference group (decomp.cpp:13-30) is then a strided walk
// in the reference's push order, so every ordered sum is unchanged, while
// the bus phase reads its rows contiguously and a branch reads two 32-byte
// quads.  Segments start on a multiple of 4; the gap after the generator
// pairs is padding (positions with no row, rid = -1, whose state stays 0).
struct RowLayout {
    int mpad = 0;                  // storage positions (>= m)
    std::vector<int> seg;          // 3 * nb: start, qstart, end
    std::vector<int> gpos;         // ng: position of the generator's p row (q at +1)
    std::vector<int> qpos;         // 2 * nl: from-quad, to-quad position of each branch
    std::vector<int> rid;          // mpad: reference row id of each position, -1 = padding
    std::vector<int> pos;          // m: position of each reference row
    std::vector<int> quad_branch;  // mpad / 4: 2 b + side of the quad at 4 q, -1 otherwise
};
RowLayout build_row_layout(const Network& net);

}  // namespace ga

#endif
