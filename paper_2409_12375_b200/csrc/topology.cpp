// xrl_topology_build: PEEC graph, CM basis maps (Algorithm 1) and the loop
// matrix (host C++, setup; SURVEY §8(a) a14-a15 inputs).
//
// panel centroids are circuit nodes, the edge shared by two panels
// is the branch between them.  Algorithm 1: A_t(e, i) =
// +rho_ie,t if rho_ie = m_e - c_i points along the branch current, else
// -rho_ie,t.  With the reference direction i -> j (i < j in library order):
//   A_t(e, i) = (m_e - c_i)_t,  A_t(e, j) = (c_j - m_e)_t.
// Loop analysis (Eq. 7): M(l, e) = +1 / -1 if branch e is
// traversed along / against its reference direction in loop l.  The paper
// defers the loop search to refs [6],[14]; this build uses (R11):
//   * one local loop around every mesh vertex (the fan of panels sharing it),
//     minus one per closed component (their sum vanishes);
//   * if those do not span the cycle space (surfaces with handles, open
//     surfaces), fundamental cycles of a BFS spanning forest instead;
//   * ports as super-nodes with zero-impedance terminal branches, terminal
//     loops through a spanning tree of each terminal set, and one port loop
//     per port (the only loop containing that port's branch).
// Loops are ordered by the Morton key of their location so that consecutive
// loops are spatially close (block-Jacobi preconditioner, a15).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <queue>

#include "xrl_internal.h"

using namespace xrl;

namespace {

struct UF {
    std::vector<int> p;
    explicit UF(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
    int f(int x) { while (p[x] != x) x = p[x] = p[p[x]]; return x; }
    void u(int a, int b) { a = f(a); b = f(b); if (a != b) p[std::max(a, b)] = std::min(a, b); }
};

uint64_t spread3h(uint32_t v)
{
    uint64_t x = v & 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

struct Loop {
    uint64_t key;                 // Morton key of its location (ordering)
    int kind;                     // 0 vertex, 1 fundamental, 2 terminal, 3 port
    std::vector<std::pair<int, int8_t>> br;  // (branch, sign)
};

}  // namespace

static xrl_status topo_impl(xrl_tree t, int32_t n_ports, const xrl_port* ports, xrl_topo* out)
{
    const int64_t n = t->n;
    cudaStream_t st = t->ctx->stream;
    XRL_CUDA(cudaSetDevice(t->ctx->device));
    auto T = std::make_unique<xrl_topo_s>();
    T->tree = t;
    // library-order geometry
    std::vector<int32_t> perm(n), iperm(n);
    std::vector<double> cent(3 * n);
    XRL_CUDA(cudaMemcpyAsync(perm.data(), t->perm.p, 4 * n, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(cent.data(), t->cent.p, 8 * 3 * n, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = (int32_t)i;
    const int64_t nv = (int64_t)t->h_vert.size() / 3;

    // ---- edges: group the 3n half-edges by vertex pair
    // (triangles: 3 half-edges; rectangle panels of hybrid meshes: 4)
    struct HE { uint64_t key; int32_t panel; };
    const int sv = t->stride;
    auto corners = [&](int64_t i, int32_t* c) {  // library panel i -> its vertex ids, count
        const int32_t* v = &t->h_tri[(int64_t)sv * perm[i]];
        c[0] = v[0]; c[1] = v[1]; c[2] = v[2];
        if (sv == 4 && v[3] >= 0) { c[3] = v[3]; return 4; }
        return 3;
    };
    std::vector<HE> he;
    he.reserve((size_t)sv * n);
    for (int64_t i = 0; i < n; ++i) {
        int32_t c[4];
        const int nc = corners(i, c);
        for (int e = 0; e < nc; ++e) {
            uint32_t a = c[e], b = c[(e + 1) % nc];
            if (a > b) std::swap(a, b);
            he.push_back({((uint64_t)a << 32) | b, (int32_t)i});
        }
    }
    std::sort(he.begin(), he.end(), [](const HE& x, const HE& y) { return x.key < y.key || (x.key == y.key && x.panel < y.panel); });
    std::vector<uint8_t> vbad(nv, 0);  // boundary or non-manifold vertex
    std::vector<uint64_t> ekey;
    for (size_t s = 0; s < he.size();) {
        size_t e = s;
        while (e < he.size() && he[e].key == he[s].key) ++e;
        const uint32_t va = (uint32_t)(he[s].key >> 32), vb = (uint32_t)(he[s].key & 0xffffffffu);
        if (e - s == 2) {
            T->edge_i.push_back(he[s].panel);
            T->edge_j.push_back(he[s + 1].panel);
            ekey.push_back(he[s].key);
        } else if (e - s > 2) {
            set_error("xrl_topology_build: non-manifold edge (%u,%u) shared by %zu panels", va, vb, e - s);
            return XRL_EGEOM;
        } else {
            vbad[va] = vbad[vb] = 1;
        }
        s = e;
    }
    const int64_t ne = (int64_t)T->edge_i.size();
    T->n_edges = ne;
    T->edge_mid.resize(3 * ne);
    for (int64_t e = 0; e < ne; ++e) {
        const uint32_t va = (uint32_t)(ekey[e] >> 32), vb = (uint32_t)(ekey[e] & 0xffffffffu);
        for (int d = 0; d < 3; ++d) T->edge_mid[3 * e + d] = 0.5 * (t->h_vert[3 * va + d] + t->h_vert[3 * vb + d]);
    }
    // branches: physical edges first
    for (int64_t e = 0; e < ne; ++e) {
        T->br_a.push_back(T->edge_i[e]);
        T->br_b.push_back(T->edge_j[e]);
        T->br_kind.push_back(0);
    }
    // components
    UF uf((int)n);
    for (int64_t e = 0; e < ne; ++e) uf.u(T->edge_i[e], T->edge_j[e]);
    std::vector<int> comp_of(n);
    int ncomp = 0;
    {
        std::vector<int> id(n, -1);
        for (int64_t i = 0; i < n; ++i) {
            int r = uf.f((int)i);
            if (id[r] < 0) id[r] = ncomp++;
            comp_of[i] = id[r];
        }
    }
    T->n_components = ncomp;
    const double invW = 1.0 / t->W;
    auto morton = [&](const double* p) {
        uint32_t q[3];
        for (int d = 0; d < 3; ++d) {
            double u = (p[d] - t->lo[d]) * invW * double(1 << 21);
            long long v = (long long)std::floor(u);
            v = std::max(0LL, std::min(v, (1LL << 21) - 1));
            q[d] = (uint32_t)v;
        }
        return spread3h(q[0]) | (spread3h(q[1]) << 1) | (spread3h(q[2]) << 2);
    };

    std::vector<Loop> loops;
    // ---- vertex loops
    std::vector<int64_t> vptr(nv + 1, 0);
    for (int64_t e = 0; e < ne; ++e) { vptr[(ekey[e] >> 32) + 1]++; vptr[(ekey[e] & 0xffffffffu) + 1]++; }
    for (int64_t v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
    std::vector<int32_t> vedge(vptr[nv]);
    {
        std::vector<int64_t> fill(vptr.begin(), vptr.end() - 1);
        for (int64_t e = 0; e < ne; ++e) {
            vedge[fill[ekey[e] >> 32]++] = (int32_t)e;
            vedge[fill[ekey[e] & 0xffffffffu]++] = (int32_t)e;
        }
    }
    std::vector<Loop> vloops;
    std::vector<int> vloop_comp;
    for (int64_t v = 0; v < nv; ++v) {
        const int64_t d = vptr[v + 1] - vptr[v];
        if (vbad[v] || d < 2) continue;
        const int32_t* E = &vedge[vptr[v]];
        // walk the fan: start at edge E[0], from panel edge_i to edge_j
        Loop L;
        L.kind = 0;
        L.key = morton(&t->h_vert[3 * v]);
        int cur_e = E[0];
        int cur_p = T->edge_j[cur_e];
        L.br.push_back({cur_e, +1});
        const int start_p = T->edge_i[cur_e];
        bool ok = true;
        for (int64_t step = 1; step <= d; ++step) {
            if (cur_p == start_p) break;
            int nxt = -1;
            for (int64_t q = 0; q < d; ++q) {
                const int e2 = E[q];
                if (e2 == cur_e) continue;
                if (T->edge_i[e2] == cur_p || T->edge_j[e2] == cur_p) { nxt = e2; break; }
            }
            if (nxt < 0) { ok = false; break; }
            const int np_ = (T->edge_i[nxt] == cur_p) ? T->edge_j[nxt] : T->edge_i[nxt];
            L.br.push_back({nxt, (int8_t)(T->edge_i[nxt] == cur_p ? +1 : -1)});
            cur_e = nxt;
            cur_p = np_;
        }
        if (!ok || cur_p != start_p || (int64_t)L.br.size() != d) continue;
        vloop_comp.push_back(comp_of[T->edge_i[E[0]]]);
        vloops.push_back(std::move(L));
    }
    // Per closed component of genus g: its vertex loops minus one (they sum
    // to zero) plus 2g handle loops span the cycle space (edges - panels + 1).
    // Handle loops by tree-cotree: BFS tree T* of the panel graph, a spanning
    // forest T of the mesh vertices over edges not crossed by T*; each of the
    // 2g remaining edges closes one fundamental cycle of T*.  Components with
    // open boundaries (or failed fans) get fundamental cycles of T* for every
    // chord instead.
    std::vector<int64_t> ecount(ncomp, 0), pcount(ncomp, 0), vcount(ncomp, 0);
    std::vector<uint8_t> comp_open(ncomp, 0);
    for (int64_t e = 0; e < ne; ++e) ecount[comp_of[T->edge_i[e]]]++;
    for (int64_t i = 0; i < n; ++i) pcount[comp_of[i]]++;
    for (size_t i = 0; i < vloops.size(); ++i) vcount[vloop_comp[i]]++;
    {
        // a component is open if any of its panels has a vertex without a closed fan
        for (int64_t i = 0; i < n; ++i) {
            int32_t c[4];
            const int nc = corners(i, c);
            for (int q = 0; q < nc; ++q)
                if (vbad[c[q]]) comp_open[comp_of[i]] = 1;
        }
        std::vector<int> last(ncomp, -1);
        for (size_t i = 0; i < vloops.size(); ++i) last[vloop_comp[i]] = (int)i;
        for (size_t i = 0; i < vloops.size(); ++i) {
            const int c = vloop_comp[i];
            if (!comp_open[c] && (int)i != last[c]) loops.push_back(std::move(vloops[i]));
        }
    }
    T->n_vertex_loops = (int64_t)loops.size();
    // adjacency of the panel graph (for BFS)
    std::vector<int64_t> pptr(n + 1, 0);
    for (int64_t e = 0; e < ne; ++e) { pptr[T->edge_i[e] + 1]++; pptr[T->edge_j[e] + 1]++; }
    for (int64_t i = 0; i < n; ++i) pptr[i + 1] += pptr[i];
    std::vector<int32_t> padj(pptr[n]);
    {
        std::vector<int64_t> fill(pptr.begin(), pptr.end() - 1);
        for (int64_t e = 0; e < ne; ++e) { padj[fill[T->edge_i[e]]++] = (int32_t)e; padj[fill[T->edge_j[e]]++] = (int32_t)e; }
    }
    auto other = [&](int e, int p) { return T->edge_i[e] == p ? T->edge_j[e] : T->edge_i[e]; };
    auto sign_from = [&](int e, int from) { return (int8_t)(T->edge_i[e] == from ? +1 : -1); };
    std::vector<uint8_t> need(ncomp, 0);  // components needing extra (handle or fundamental) loops
    bool any = false;
    for (int c = 0; c < ncomp; ++c) {
        const int64_t rank_c = ecount[c] - pcount[c] + 1;
        need[c] = comp_open[c] || (vcount[c] - 1 != rank_c);
        any = any || need[c];
    }
    if (any) {
        // BFS tree T* of the panel graph in those components
        std::vector<int> par_e(n, -1), depth(n, -1);
        for (int64_t r = 0; r < n; ++r) {
            if (depth[r] >= 0 || !need[comp_of[r]]) continue;
            std::queue<int> q;
            q.push((int)r);
            depth[r] = 0;
            while (!q.empty()) {
                int p = q.front(); q.pop();
                for (int64_t k = pptr[p]; k < pptr[p + 1]; ++k) {
                    int e = padj[k], o = other(e, p);
                    if (depth[o] < 0) { depth[o] = depth[p] + 1; par_e[o] = e; q.push(o); }
                }
            }
        }
        std::vector<uint8_t> in_tstar(ne, 0);
        for (int64_t i = 0; i < n; ++i)
            if (par_e[i] >= 0) in_tstar[par_e[i]] = 1;
        // closed components: spanning forest T of the vertices over edges not in T*
        std::vector<uint8_t> in_t(ne, 0);
        {
            UF vuf((int)nv);
            for (int64_t e = 0; e < ne; ++e) {
                const int c = comp_of[T->edge_i[e]];
                if (!need[c] || comp_open[c] || in_tstar[e]) continue;
                const int va = (int)(ekey[e] >> 32), vb = (int)(ekey[e] & 0xffffffffu);
                if (vuf.f(va) != vuf.f(vb)) { vuf.u(va, vb); in_t[e] = 1; }
            }
        }
        for (int64_t e = 0; e < ne; ++e) {
            int a = T->edge_i[e], b = T->edge_j[e];
            const int c = comp_of[a];
            if (!need[c] || in_tstar[e]) continue;
            if (!comp_open[c] && in_t[e]) continue;  // closed: only the 2g leftover chords
            Loop L;
            L.kind = 1;
            L.key = morton(&T->edge_mid[3 * e]);
            // chord a -> b, then tree path b -> a
            L.br.push_back({(int)e, +1});
            std::vector<std::pair<int, int8_t>> up_b, up_a;
            int x = b, y = a;
            while (x != y) {
                if (depth[x] >= depth[y]) { int pe = par_e[x]; int px = other(pe, x); up_b.push_back({pe, sign_from(pe, x)}); x = px; }
                else { int pe = par_e[y]; int py = other(pe, y); up_a.push_back({pe, sign_from(pe, py)}); y = py; }
            }
            for (auto& z : up_b) L.br.push_back(z);
            for (auto it = up_a.rbegin(); it != up_a.rend(); ++it) L.br.push_back(*it);
            loops.push_back(std::move(L));
        }
    }
    T->n_fund_loops = (int64_t)loops.size() - T->n_vertex_loops;
    std::sort(loops.begin(), loops.end(), [](const Loop& a, const Loop& b) { return a.key < b.key; });

    // ---- ports
    const int64_t nsuper0 = n;
    auto bfs_path = [&](int from, const std::vector<uint8_t>& target, std::vector<std::pair<int, int8_t>>& path) -> int {
        std::vector<int> pe(n, -2);
        std::queue<int> q;
        q.push(from);
        pe[from] = -1;
        int hit = -1;
        while (!q.empty() && hit < 0) {
            int p = q.front(); q.pop();
            if (target[p]) { hit = p; break; }
            for (int64_t k = pptr[p]; k < pptr[p + 1]; ++k) {
                int e = padj[k], o = other(e, p);
                if (pe[o] == -2) { pe[o] = e; q.push(o); }
            }
        }
        if (hit < 0) return -1;
        std::vector<std::pair<int, int8_t>> rev;
        for (int x = hit; x != from;) { int e = pe[x]; int px = other(e, x); rev.push_back({e, sign_from(e, px)}); x = px; }
        path.assign(rev.rbegin(), rev.rend());
        return hit;
    };
    std::vector<Loop> tloops, ploops;
    for (int p = 0; p < n_ports; ++p) {
        const int Sp = (int)(nsuper0 + 2 * p), Sm = Sp + 1;
        std::vector<int> setP, setM;
        for (int s = 0; s < 2; ++s) {
            const int32_t* ids = s == 0 ? ports[p].plus : ports[p].minus;
            const int cnt = s == 0 ? ports[p].n_plus : ports[p].n_minus;
            if (cnt < 1 || !ids) { set_error("xrl_topology_build: port %d has an empty terminal", p); return XRL_EINVAL; }
            for (int k = 0; k < cnt; ++k) {
                if (ids[k] < 0 || ids[k] >= n) { set_error("xrl_topology_build: port %d panel id out of range", p); return XRL_EINVAL; }
                (s == 0 ? setP : setM).push_back(iperm[ids[k]]);
            }
        }
        // terminal branches
        std::vector<int> brP(n, -1), brM(n, -1);
        for (int k : setP) { brP[k] = (int)T->br_a.size(); T->br_a.push_back(Sp); T->br_b.push_back(k); T->br_kind.push_back(1); }
        for (int k : setM) { brM[k] = (int)T->br_a.size(); T->br_a.push_back(k); T->br_b.push_back(Sm); T->br_kind.push_back(1); }
        const int bport = (int)T->br_a.size();
        T->br_a.push_back(Sm); T->br_b.push_back(Sp); T->br_kind.push_back(2);
        // terminal loops: spanning tree of each terminal set (paths through the panel graph)
        for (int s = 0; s < 2; ++s) {
            std::vector<int>& S = s == 0 ? setP : setM;
            std::vector<uint8_t> in(n, 0), done(n, 0);
            for (int k : S) in[k] = 1;
            const int root = S[0];
            done[root] = 1;
            for (size_t a = 1; a < S.size(); ++a) {
                const int k = S[a];
                if (done[k]) continue;
                std::vector<uint8_t> tgt(n, 0);
                tgt[k] = 1;
                std::vector<std::pair<int, int8_t>> path;
                if (bfs_path(root, tgt, path) < 0) { set_error("xrl_topology_build: port %d terminal not connected", p); return XRL_EGEOM; }
                Loop L;
                L.kind = 2;
                L.key = ~0ull;
                if (s == 0) {  // Sp -> root, path root -> k, k -> Sp (against Sp->k)
                    L.br.push_back({brP[root], +1});
                    for (auto& z : path) L.br.push_back(z);
                    L.br.push_back({brP[k], -1});
                } else {       // root -> k (path), k -> Sm, Sm -> root (against root->Sm)
                    for (auto& z : path) L.br.push_back(z);
                    L.br.push_back({brM[k], +1});
                    L.br.push_back({brM[root], -1});
                }
                done[k] = 1;
                tloops.push_back(std::move(L));
            }
        }
        // port loop: Sm -> Sp (port branch), Sp -> k+, path k+ -> k-, k- -> Sm
        std::vector<uint8_t> tgtM(n, 0);
        for (int k : setM) tgtM[k] = 1;
        std::vector<std::pair<int, int8_t>> path;
        const int hit = bfs_path(setP[0], tgtM, path);
        if (hit < 0) { set_error("xrl_topology_build: port %d terminals are disconnected", p); return XRL_EGEOM; }
        Loop L;
        L.kind = 3;
        L.key = ~0ull;
        L.br.push_back({bport, +1});
        L.br.push_back({brP[setP[0]], +1});
        for (auto& z : path) L.br.push_back(z);
        L.br.push_back({brM[hit], +1});
        ploops.push_back(std::move(L));
    }
    T->n_terminal_loops = (int64_t)tloops.size();
    for (auto& L : tloops) loops.push_back(std::move(L));
    for (int p = 0; p < n_ports; ++p) {
        T->port_loop.push_back((int32_t)loops.size());
        loops.push_back(std::move(ploops[p]));
    }
    T->n_ports = n_ports;
    T->n_branches = (int64_t)T->br_a.size();
    T->n_loops = (int64_t)loops.size();
    T->loop_kind.resize(T->n_loops);
    // M CSR
    T->m_ptr.assign(T->n_loops + 1, 0);
    for (int64_t l = 0; l < T->n_loops; ++l) {
        T->loop_kind[l] = (int8_t)loops[l].kind;
        T->m_ptr[l + 1] = T->m_ptr[l] + (int64_t)loops[l].br.size();
        for (auto& z : loops[l].br) { T->m_idx.push_back(z.first); T->m_val.push_back(z.second); }
    }
    // C = (M A_t) restricted to physical edges: loop rows, panel columns, 3 values
    std::vector<int64_t> clp(T->n_loops + 1, 0);
    std::vector<int32_t> clc;
    std::vector<double> clv;
    for (int64_t l = 0; l < T->n_loops; ++l) {
        std::vector<std::pair<int32_t, std::array<double, 3>>> ent;
        for (auto& z : loops[l].br) {
            const int b = z.first;
            if (T->br_kind[b] != 0) continue;
            const double s = z.second;
            const int i = T->edge_i[b], j = T->edge_j[b];
            const double* m = &T->edge_mid[3 * b];
            ent.push_back({i, {s * (m[0] - cent[3 * i]), s * (m[1] - cent[3 * i + 1]), s * (m[2] - cent[3 * i + 2])}});
            ent.push_back({j, {s * (cent[3 * j] - m[0]), s * (cent[3 * j + 1] - m[1]), s * (cent[3 * j + 2] - m[2])}});
        }
        std::sort(ent.begin(), ent.end(), [](auto& a, auto& b) { return a.first < b.first; });
        for (size_t a = 0; a < ent.size();) {
            size_t b = a;
            std::array<double, 3> acc{0, 0, 0};
            while (b < ent.size() && ent[b].first == ent[a].first) { for (int d = 0; d < 3; ++d) acc[d] += ent[b].second[d]; ++b; }
            clc.push_back(ent[a].first);
            for (int d = 0; d < 3; ++d) clv.push_back(acc[d]);
            a = b;
        }
        clp[l + 1] = (int64_t)clc.size();
    }
    T->nnz_c = (int64_t)clc.size();
    T->c_ptr_h = clp;
    T->c_col_h = clc;
    T->c_val_h = clv;
    // transpose: panel rows, loop columns
    std::vector<int64_t> cpp(n + 1, 0);
    for (int32_t c : clc) cpp[c + 1]++;
    for (int64_t i = 0; i < n; ++i) cpp[i + 1] += cpp[i];
    std::vector<int32_t> cpc(clc.size());
    std::vector<float> cpv(3 * clc.size());
    std::vector<double> cpv64(3 * clc.size());
    {
        std::vector<int64_t> fill(cpp.begin(), cpp.end() - 1);
        for (int64_t l = 0; l < T->n_loops; ++l)
            for (int64_t q = clp[l]; q < clp[l + 1]; ++q) {
                const int64_t o = fill[clc[q]]++;
                cpc[o] = (int32_t)l;
                for (int d = 0; d < 3; ++d) {
                    cpv[3 * o + d] = (float)clv[3 * q + d];
                    cpv64[3 * o + d] = clv[3 * q + d];
                }
            }
    }
    std::vector<float> clvf(clv.begin(), clv.end());
    T->cl_ptr.alloc(T->n_loops + 1);
    T->cl_col.alloc(std::max<size_t>(1, clc.size()));
    T->cl_val.alloc(std::max<size_t>(3, clvf.size()));
    T->cl_val64.alloc(std::max<size_t>(3, clv.size()));
    T->cp_ptr.alloc(n + 1);
    T->cp_col.alloc(std::max<size_t>(1, cpc.size()));
    T->cp_val.alloc(std::max<size_t>(3, cpv.size()));
    T->cp_val64.alloc(std::max<size_t>(3, cpv64.size()));
    XRL_CUDA(cudaMemcpyAsync(T->cl_ptr.p, clp.data(), 8 * clp.size(), cudaMemcpyHostToDevice, st));
    if (!clc.empty()) {
        XRL_CUDA(cudaMemcpyAsync(T->cl_col.p, clc.data(), 4 * clc.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->cl_val.p, clvf.data(), 4 * clvf.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->cl_val64.p, clv.data(), 8 * clv.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->cp_col.p, cpc.data(), 4 * cpc.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->cp_val.p, cpv.data(), 4 * cpv.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->cp_val64.p, cpv64.data(), 8 * cpv64.size(), cudaMemcpyHostToDevice, st));
    }
    XRL_CUDA(cudaMemcpyAsync(T->cp_ptr.p, cpp.data(), 8 * cpp.size(), cudaMemcpyHostToDevice, st));
    {
        std::vector<int32_t> lr;
        for (int64_t l = 0; l < T->n_loops; ++l)
            if (clp[l + 1] - clp[l] > 64) lr.push_back((int32_t)l);
        T->n_long = (int32_t)lr.size();
        T->long_rows.alloc(std::max<size_t>(1, lr.size()));
        if (!lr.empty()) XRL_CUDA(cudaMemcpyAsync(T->long_rows.p, lr.data(), 4 * lr.size(), cudaMemcpyHostToDevice, st));
    }
    XRL_CUDA(cudaStreamSynchronize(st));
    T->perm = perm;
    ++t->refs;
    *out = T.release();
    return XRL_OK;
}

void xrl::topo_release(xrl_topo T)
{
    if (!T->dead || T->refs > 0) return;
    xrl_tree t = T->tree;
    delete T;
    --t->refs;
    tree_release(t);
}

extern "C" {

xrl_status xrl_topology_build(xrl_tree t, int32_t n_ports, const xrl_port* ports, xrl_topo* out)
{
    if (!t || !out || n_ports < 0 || (n_ports > 0 && !ports)) { set_error("xrl_topology_build: bad argument"); return XRL_EINVAL; }
    *out = nullptr;

    try {
        return topo_impl(t, n_ports, ports, out);
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return XRL_ENOMEM;
    }
}

void xrl_topology_destroy(xrl_topo T)
{
    if (!T) return;
    T->dead = true;
    topo_release(T);  // deferred while operators built on it are alive
}

xrl_status xrl_topology_info(xrl_topo T, xrl_topo_info_t* info)
{
    if (!T || !info) { set_error("xrl_topology_info: null argument"); return XRL_EINVAL; }
    info->n_panels = T->tree->n;
    info->n_edges = T->n_edges;
    info->n_branches = T->n_branches;
    info->n_loops = T->n_loops;
    info->n_ports = T->n_ports;
    info->n_components = T->n_components;
    info->n_vertex_loops = T->n_vertex_loops;
    info->n_fundamental_loops = T->n_fund_loops;
    info->n_terminal_loops = T->n_terminal_loops;
    info->nnz_m = (int64_t)T->m_idx.size();
    info->nnz_c = T->nnz_c;
    return XRL_OK;
}

xrl_status xrl_topology_export(xrl_topo T, int32_t* branch_nodes, int8_t* branch_kind, double* edge_mid,
                               int64_t* m_ptr, int32_t* m_branch, int8_t* m_sign, int32_t* port_loop, int8_t* loop_kind,
                               int64_t* c_ptr, int32_t* c_panel, double* c_val)
{
    if (!T) { set_error("xrl_topology_export: null handle"); return XRL_EINVAL; }
    const int64_t n = T->tree->n;
    if (branch_nodes)
        for (int64_t b = 0; b < T->n_branches; ++b) {
            auto node = [&](int x) -> int32_t { return x < n ? T->perm[x] : (int32_t)(-1 - (x - n)); };
            branch_nodes[2 * b] = node(T->br_a[b]);
            branch_nodes[2 * b + 1] = node(T->br_b[b]);
        }
    if (branch_kind) std::copy(T->br_kind.begin(), T->br_kind.end(), branch_kind);
    if (edge_mid) std::copy(T->edge_mid.begin(), T->edge_mid.end(), edge_mid);
    if (m_ptr) std::copy(T->m_ptr.begin(), T->m_ptr.end(), m_ptr);
    if (m_branch) std::copy(T->m_idx.begin(), T->m_idx.end(), m_branch);
    if (m_sign) std::copy(T->m_val.begin(), T->m_val.end(), m_sign);
    if (port_loop) std::copy(T->port_loop.begin(), T->port_loop.end(), port_loop);
    if (loop_kind) std::copy(T->loop_kind.begin(), T->loop_kind.end(), loop_kind);
    if (c_ptr) std::copy(T->c_ptr_h.begin(), T->c_ptr_h.end(), c_ptr);
    if (c_panel)
        for (size_t q = 0; q < T->c_col_h.size(); ++q) c_panel[q] = T->perm[T->c_col_h[q]];
    if (c_val) std::copy(T->c_val_h.begin(), T->c_val_h.end(), c_val);
    return XRL_OK;
}

}  // extern "C"
