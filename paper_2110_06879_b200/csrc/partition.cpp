// partition.cpp — see partition.hpp.
#include "partition.hpp"

#include <algorithm>
#include <queue>

namespace ga {

std::vector<int> partition_buses(const Network& net, int k) {
    const int nb = net.nb(), nl = net.nl();
    std::vector<int> part(nb, 0);
    if (k <= 1 || nb == 0) return part;
    // adjacency in ascending neighbour order
    std::vector<std::vector<int>> adj(nb);
    std::vector<long long> weight(nb, 1);
    const bool measured = static_cast<int>(net.branch_weight.size()) == nl;
    for (int b = 0; b < nl; ++b) {
        const int f = net.lines[b].from, t = net.lines[b].to;
        adj[f].push_back(t);
        adj[t].push_back(f);
        // a branch is solved on its from-bus part (the dominant work).  With
        // measured weights (TRON steps of a previous sweep) the heavy-tailed
        // branches spread over the parts; otherwise a rate-limited branch (6
        // variables + the AL loop) costs about twice an unlimited one per
        // TRON iteration (census) and runs the AL tails
        if (measured) weight[f] += 1 + static_cast<long long>(net.branch_weight[b]);
        else weight[f] += net.lines[b].limited() ? 8 : 4;
    }
    for (auto& a : adj) std::sort(a.begin(), a.end());
    std::vector<int> order;
    order.reserve(nb);
    std::vector<char> seen(nb, 0);
    for (int s = 0; s < nb; ++s) {  // all components, BFS each
        if (seen[s]) continue;
        std::queue<int> q;
        q.push(s);
        seen[s] = 1;
        while (!q.empty()) {
            const int u = q.front();
            q.pop();
            order.push_back(u);
            for (int v : adj[u])
                if (!seen[v]) {
                    seen[v] = 1;
                    q.push(v);
                }
        }
    }
    long long total = 0;
    for (long long w : weight) total += w;
    long long acc = 0;
    for (int u : order) {
        int p = static_cast<int>((acc * k) / std::max<long long>(total, 1));
        part[u] = std::min(p, k - 1);
        acc += weight[u];
    }
    return part;
}

PartPlan make_plan(const Network& net, const std::vector<int>& part, int p, int k) {
    PartPlan pl;
    // k parts as requested, whether or not the partition left some empty
    k = std::max({k, 1, part.empty() ? 1 : 1 + *std::max_element(part.begin(), part.end())});
    pl.part = p;
    pl.parts = k;
    pl.send_x.assign(k, {});
    pl.recv_x.assign(k, {});
    const int ng = net.ng(), nl = net.nl(), nb = net.nb();
    for (int i = 0; i < nb; ++i)
        if (part[i] == p) pl.buses.push_back(i);
    std::vector<char> own_row(static_cast<size_t>(net.m()), 0);
    for (int g = 0; g < ng; ++g)
        if (part[net.gens[g].bus] == p) {
            pl.gens.push_back(g);
            own_row[2 * g] = own_row[2 * g + 1] = 1;
        }
    static const int kFrom[4] = {0, 1, 4, 5}, kTo[4] = {2, 3, 6, 7};
    for (int b = 0; b < nl; ++b) {
        const int pf = part[net.lines[b].from], pt = part[net.lines[b].to];
        const int base = 2 * ng + 8 * b;
        if (pf == p) {
            (net.lines[b].limited() ? pl.lim : pl.unl).push_back(b);
            for (int k4 : kFrom) own_row[base + k4] = 1;
        }
        if (pt == p)
            for (int k4 : kTo) own_row[base + k4] = 1;
        if (pf == p && pt != p)
            for (int k4 : kTo) pl.send_x[pt].push_back(base + k4);
        if (pt == p && pf != p)
            for (int k4 : kTo) pl.recv_x[pf].push_back(base + k4);
    }
    for (int r = 0; r < net.m(); ++r)
        if (own_row[r]) pl.rows.push_back(r);
    return pl;
}

}  // namespace ga
