// pf_graph.cu -- label-graph compilation (row a10; reading R9).
#include "pf_internal.h"

namespace pfi {

pf_status compile_graph(const pf_graph *gr, Compiled *out) {
    if (!gr || gr->num_nodes < 3 || gr->num_edges < 2 || !gr->parent || !gr->child || !gr->weight)
        return fail(PF_ERR_GRAPH, "graph: need >= 3 nodes (S + 2 end labels), >= 2 edges and non-NULL arrays");
    const int n = gr->num_nodes, ne = gr->num_edges;
    std::string errs;
    auto add = [&](const std::string &s) { errs += (errs.empty() ? "" : "; ") + s; };
    std::vector<std::vector<std::pair<int, float>>> kids(n), pars(n);
    bool idx_ok = true;
    for (int e = 0; e < ne; ++e) {
        const int p = gr->parent[e], c = gr->child[e];
        const float w = gr->weight[e];
        if (p < 0 || p >= n || c < 0 || c >= n) {
            add("edge " + std::to_string(e) + " has a node id out of range");
            idx_ok = false;
            continue;
        }
        if (!(w > 0.f) || !std::isfinite(w)) add("edge " + std::to_string(e) + " weight must be > 0");
        if (p == c) add("self-loop at node " + std::to_string(p));
        kids[p].push_back({c, w});
        pars[c].push_back({p, w});
    }
    if (!idx_ok) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    if (!pars[0].empty()) add("source S (node 0) has parents");
    // Kahn with lowest-id tie-break
    std::vector<int> indeg(n, 0), order;
    for (int v = 0; v < n; ++v) indeg[v] = (int)pars[v].size();
    std::vector<bool> placed(n, false);
    for (int k = 0; k < n; ++k) {
        int pick = -1;
        for (int v = 0; v < n; ++v)
            if (!placed[v] && indeg[v] == 0) { pick = v; break; }
        if (pick < 0) break;
        placed[pick] = true;
        order.push_back(pick);
        for (auto &c : kids[pick]) indeg[c.first]--;
    }
    if ((int)order.size() != n) add("graph has a cycle");
    // reachability from S
    std::vector<bool> reach(n, false);
    std::vector<int> stack{0};
    reach[0] = true;
    while (!stack.empty()) {
        int v = stack.back();
        stack.pop_back();
        for (auto &c : kids[v])
            if (!reach[c.first]) { reach[c.first] = true; stack.push_back(c.first); }
    }
    for (int v = 1; v < n; ++v)
        if (!reach[v]) add("node " + std::to_string(v) + " unreachable from S");
    std::vector<int> leaves, internals;
    for (int v = 1; v < n; ++v) (kids[v].empty() ? leaves : internals).push_back(v);
    if (leaves.size() < 2) add("fewer than 2 end labels");
    if (!errs.empty()) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    // W_(v, B) by memoised recursion in reverse topological order
    const int NL = (int)leaves.size();
    std::vector<std::vector<double>> Wd(n, std::vector<double>(NL, 0.0));
    for (int k = n - 1; k >= 0; --k) {
        const int v = order[k];
        if (kids[v].empty() && v != 0) {
            Wd[v][std::find(leaves.begin(), leaves.end(), v) - leaves.begin()] = 1.0;
        } else {
            for (auto &c : kids[v])
                for (int l = 0; l < NL; ++l) Wd[v][l] += (double)c.second * Wd[c.first][l];
        }
    }
    for (int l = 0; l < NL; ++l)
        if (std::fabs(Wd[0][l] - 1.0) > 1e-6)
            add("W_(S," + std::to_string(leaves[l]) + ") = " + std::to_string(Wd[0][l]) +
                " != 1 (sum of end labels must equal u_S = 1, reading R9)");
    if (!errs.empty()) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    const int NI = (int)internals.size();
    // Ishikawa chain: internals in topological order N_1..N_N, S -> {N_1, L_0}, N_i -> {N_{i+1}, L_i},
    // N_N -> L_N, all weights 1, end labels in increasing id order L_0..L_N
    bool chain = NL == NI + 1 && NI >= 1 && kids[0].size() == 2;
    std::vector<int> lev;
    for (int k = 0; k < n && chain; ++k)
        if (order[k] != 0 && !kids[order[k]].empty()) lev.push_back(order[k]);
    auto has_edge = [&](int p, int c) {
        for (auto &e : kids[p])
            if (e.first == c && e.second == 1.f) return true;
        return false;
    };
    if (chain) {
        chain = (int)lev.size() == NI && has_edge(0, lev[0]) && has_edge(0, leaves[0]);
        for (int i = 0; i < NI && chain; ++i) {
            const bool last = i == NI - 1;
            chain = kids[lev[i]].size() == (last ? 1u : 2u) && has_edge(lev[i], leaves[i + 1]) &&
                    (last || has_edge(lev[i], lev[i + 1]));
        }
    }
    // graphs beyond the compiled kernel set (<= kMaxInternal internal, <= kMaxNodes non-source nodes) run on the
    // generic path (pf_generic.cu) up to kWideNodes non-source nodes and 16 end labels
    if (NI + NL > kWideNodes || NL > 16)
        return fail(PF_ERR_UNSUPPORTED, "graph: %d internal + %d end nodes exceeds the supported size "
                                        "(<= %d non-source nodes, <= 16 end labels)", NI, NL, kWideNodes);
    if (chain && NL > kMaxNodes)
        return fail(PF_ERR_UNSUPPORTED, "graph: Ishikawa chain with %d labels exceeds %d", NL, kMaxNodes);
    out->chain = chain;
    out->num_nodes = n;
    out->NI = NI;
    out->NL = NL;
    out->NV = NI + NL;
    out->pos_of_node.assign(n, -1);
    out->node_of_pos.clear();
    for (int k = 0; k < n; ++k) {  // internal nodes in topological order
        const int v = order[k];
        if (v != 0 && !kids[v].empty()) {
            out->pos_of_node[v] = (int)out->node_of_pos.size();
            out->node_of_pos.push_back(v);
        }
    }
    for (int v : leaves) {  // end labels in node-id order
        out->pos_of_node[v] = (int)out->node_of_pos.size();
        out->node_of_pos.push_back(v);
    }
    memset(&out->g, 0, sizeof(out->g));
    memset(&out->gw, 0, sizeof(out->gw));
    for (int v = 1; v < n; ++v) {  // dense weights (unused by the chain kernels)
        if (kids[v].empty()) continue;
        const int i = out->pos_of_node[v];
        for (auto &c : kids[v]) {
            const int j = out->pos_of_node[c.first];
            out->gw.w[i][j] += c.second;
            if (NI <= kMaxInternal && NI + NL <= kMaxNodes) out->g.w[i][j] += c.second;
        }
    }
    out->w_src.assign(out->NV, 0.f);
    for (auto &c : kids[0]) out->w_src[out->pos_of_node[c.first]] += c.second;
    out->W.assign(out->NV, std::vector<float>(NL, 0.f));  // W_(v, B), for reports
    for (int p = 0; p < out->NV; ++p)
        for (int l = 0; l < NL; ++l) out->W[p][l] = (float)Wd[out->node_of_pos[p]][l];
    return PF_OK;
}

}  // namespace pfi
