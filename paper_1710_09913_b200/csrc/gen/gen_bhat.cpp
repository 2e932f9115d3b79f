// gen_bhat.cpp -- build-time generator of the apply kernel's element body.
//
// For every (d, p, form) with d in {2,3}, p in 1..4 it emits a straight-line
// device function computing, for one element, Algorithm 1's line 4
// (transpose per reading L8):
//     g = Bhat u_T,  h = A_T g,  y_T += Bhat^T h
// node by node over the double-grid nodes j (so only u_T and y_T live in
// registers), from the EXACT sparse Bhat of host/tables.hpp: zero entries are
// skipped, +-1 entries become adds/subtracts (the paper's nnz_{+-1} saving,
// eq:comp_eff P:548), all other entries are fp64 FMAs with correctly rounded
// literals.  Weights are read through the policy object `pol.w(k)` with a
// compile-time row k = j * NC + c, and `pol.begin<j>() / pol.end<j>()`
// bracket each node so the kernel can pipeline the weight stream.
//
// Usage: gen_bhat <output.cuh>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "../host/tables.hpp"

using namespace dogip;

static std::string lit(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    std::string s(buf);
    if (s.find('.') == std::string::npos && s.find('e') == std::string::npos && s.find("inf") == std::string::npos)
        s += ".0";
    return s;
}

static int g_split = 0;   // rows with >= g_split terms use two interleaved partial sums (argv[3]; 0 = off)

// symmetry-adapted bodies read v through DOGIP_SYM_V(k, slot) (src "V"): registers by default,
// or the u_T staging slot `slot` in shared memory (DOGIP_SYM_VSMEM A/B builds)
static const std::vector<int>* g_vslot = nullptr;

static std::string chain(const std::vector<std::pair<int, Rat>>& terms, const char* src, int& flops) {
    bool first = true;
    std::string acc;   // a chain of fma for determinism and contraction control
    for (auto& t : terms) {
        const std::string src_l = (std::string(src) == "V" && g_vslot)
            ? "DOGIP_SYM_V(" + std::to_string(t.first) + ", " + std::to_string((*g_vslot)[t.first]) + ")"
            : std::string(src) + "[" + std::to_string(t.first) + "]";
        const Rat& c = t.second;
        if (first) {
            if (c == Rat(1)) acc = src_l;
            else if (c == Rat(-1)) acc = "-" + src_l;
            else { acc = lit(c.to_double()) + " * " + src_l; flops += 1; }
            first = false;
        } else {
            if (c == Rat(1)) acc = "(" + acc + ") + " + src_l;
            else if (c == Rat(-1)) acc = "(" + acc + ") - " + src_l;
            else { acc = "__fma_rn(" + lit(c.to_double()) + ", " + src_l + ", " + acc + ")"; flops += 1; }
            flops += 1;
        }
    }
    return acc;
}

// emit "dst = sum_l c_l src[l]" for a sparse row; returns flop count
static int emit_combo(FILE* f, const char* indent, const std::string& dst, bool declare,
                      const std::vector<std::pair<int, Rat>>& terms, const char* src) {
    int flops = 0;
    if (terms.empty()) {
        std::fprintf(f, "%s%s%s = 0.0;\n", indent, declare ? "const double " : "", dst.c_str());
        return 0;
    }
    if (g_split > 0 && (int)terms.size() >= g_split) {
        // two independent half-chains (even / odd terms) joined by one add: more ILP
        std::vector<std::pair<int, Rat>> a, b;
        for (size_t i = 0; i < terms.size(); ++i) (i % 2 ? b : a).push_back(terms[i]);
        const std::string ea = chain(a, src, flops), eb = chain(b, src, flops);
        flops += 1;
        std::fprintf(f, "%s%s%s = (%s) + (%s);\n", indent, declare ? "const double " : "", dst.c_str(), ea.c_str(),
                     eb.c_str());
        return flops;
    }
    const std::string acc = chain(terms, src, flops);
    std::fprintf(f, "%s%s%s = %s;\n", indent, declare ? "const double " : "", dst.c_str(), acc.c_str());
    return flops;
}

// One storage variant of one (d, p, form):
//   STORE 0 (full)  rows per node NC = 1 (WP) or d(d+1)/2 (EL upper triangle of A_{T,j})
//   STORE 1 (iso)   EL with isotropic M = m I (Corollary, element-wise):
//                   A_{T,j} = a_{T,j} G_T, G_T = Rinv Rinv^T; NG = d(d+1)/2 leading
//                   rows hold G_T, then one row a_{T,j} per node.
// interpolated values per emission group (argv[2]); 1 = node by node, which measured
// best on B200 (profiles/r01_ab_variants.log: grouping 12 values was neutral-to-worse)
static int g_gmax_vals = 1;
// EL bodies through the barycentric derivatives (argv[6]: bit 0 interpolation, bit 1
// projection (3D; bit 2 also 2D); default 2): per node
//   t_i = sum_l D_i[j,l] u_l (i = 0..d),  g_r = t_{r+1} - t_0,
//   y_l += sum_{i>=1} D_i[j,l] h_{i-1} - D_0[j,l] (h_0 + .. + h_{d-1})
// = the Bhat_EL body exactly (Bhat_r = D_{r+1} - D_0), with 3D P3 740 instead of 1014
// table nonzeros per direction (tables.hpp bary_deriv_table).
static int g_bary = 2;   // default: projection only, 3D only (profiles/r01_ab_bary_deriv.log:
                         // the interpolation half spills at 168 registers; 2D measured 1-2 % slower)

static void emit_variant(FILE* f, int d, int p, int form, int store) {
    Table t = bhat_table(d, p, form);
    const int VT = t.cols, WT = t.rows;
    const bool bary = form == 1 && (g_bary & 1), bary_p = form == 1 && (g_bary & 2) && (d == 3 || (g_bary & 4));
    const bool bary_any = bary || bary_p;
    Table D;
    if (bary_any) D = bary_deriv_table(d, p);
    const int NSYM = d * (d + 1) / 2;
    const int NC = (form == 0 || store == 1) ? 1 : NSYM;
    const int NG = store == 1 ? NSYM : 0;
    const int ROWS = 12;                                   // rows per streamed chunk (3 KB / warp)
    const int TILE_ROWS = NG + WT * NC;
    int nnz = 0, pm1 = 0;
    for (auto& v : t.v) { nnz += !v.is_zero(); pm1 += v.is_pm1(); }
    auto simp = cell_simplices(d);
    auto A = multi_indices(d, p);
    std::fprintf(f, "template <> struct RefElem<%d, %d, %d, %d> {\n", d, p, form, store);
    std::fprintf(f, "    static constexpr int VT = %d, WT = %d, NC = %d, NG = %d, ROWS = %d, TILE_ROWS = %d, NS = %d, RALIGN = %d, PAIR = 0, DOT_IN_BODY = 0, HAS_ROWPERM = 0;\n",
                 VT, WT, NC, NG, ROWS, TILE_ROWS, (int)simp.size(), NC);
    std::fprintf(f, "    static constexpr int NNZ = %d, NNZ_PM1 = %d;\n", nnz, pm1);
    std::fprintf(f, "    static constexpr signed char LOFF[%d][%d][%d] = {", (int)simp.size(), VT, d);
    for (size_t s = 0; s < simp.size(); ++s) {
        std::fprintf(f, "%s{", s ? ", " : "");
        for (int l = 0; l < VT; ++l) {
            std::fprintf(f, "%s{", l ? "," : "");
            for (int ax = 0; ax < d; ++ax) {
                int o = 0;
                for (int i = 0; i <= d; ++i) o += A[l][i] * simp[s][i][ax];
                std::fprintf(f, "%s%d", ax ? "," : "", o);
            }
            std::fprintf(f, "}");
        }
        std::fprintf(f, "}");
    }
    std::fprintf(f, "};\n");
    // ALPHA[l][i-1] = alpha_i of local DoF l (i = 1..d).  Every simplex of the cell has
    // v_0 = cell origin, so LOFF[s][l] = sum_i ALPHA[l][i-1] * v_i(s): the kernel forms
    // gather offsets from d per-tile vertex strides instead of a per-DoF table.
    for (auto& sv : simp)
        if (sv[0][0] || sv[0][1] || sv[0][2]) { std::fprintf(stderr, "v_0 must be the cell origin\n"); std::exit(1); }
    std::fprintf(f, "    static constexpr signed char ALPHA[%d][3] = {", VT);
    for (int l = 0; l < VT; ++l)
        std::fprintf(f, "%s{%d,%d,%d}", l ? "," : "", A[l][1], A[l][2], d == 3 ? A[l][3] : 0);
    std::fprintf(f, "};\n");
    // row of node j's first weight, and its chunk
    auto row = [&](int j) { return NG + j * NC; };
    auto chunk = [&](int j) { return row(j) / ROWS; };
    std::fprintf(f, "    static __host__ __device__ constexpr int row_of(int j) { return %d + j * %d; }\n", NG, NC);
    std::fprintf(f,
        "    template <class Pol>\n"
        "    static __device__ __forceinline__ void body(const double* __restrict__ u,\n"
        "                                                double* __restrict__ y, Pol& pol) {\n");
    int flops = 0;
    int idx[3][3], c = 0;
    for (int r = 0; r < d; ++r)
        for (int s2 = r; s2 < d; ++s2) { idx[r][s2] = idx[s2][r] = c++; }
    // Nodes are emitted in groups = the nodes whose weights share one streamed chunk:
    // all interpolations of a group first (independent FMA chains -> ILP), then weight
    // multiply + projection node by node.
    if (store == 1) {   // G_T rows lead the first chunk: open it, keep G_T in registers
        std::fprintf(f, "        pol.template begin<0>();\n");
        for (int k = 0; k < NG; ++k) std::fprintf(f, "        const double G%d = pol.w(%d);\n", k, k);
    }
    for (int j0 = 0; j0 < WT;) {
        // a group never spans a chunk and holds at most 12 interpolated values
        const int gmax = std::max(1, g_gmax_vals / t.nblk);
        int j1 = j0;
        while (j1 < WT && chunk(j1) == chunk(j0) && j1 - j0 < gmax) ++j1;
        std::fprintf(f, "        {\n");
        for (int j = j0; j < j1; ++j)
            if (!(store == 1 && j == 0)) std::fprintf(f, "          pol.template begin<%d>();\n", j);
        for (int j = j0; j < j1; ++j) {
            if (bary) {
                const std::string sj = "_" + std::to_string(j);
                bool t0 = false;
                for (int i = 0; i <= d; ++i) {
                    std::vector<std::pair<int, Rat>> terms;
                    for (int l = 0; l < VT; ++l)
                        if (!D.at(i, j, l).is_zero()) terms.push_back({l, D.at(i, j, l)});
                    if (i == 0) t0 = !terms.empty();
                    flops += emit_combo(f, "          ", "t" + std::to_string(i) + "b" + sj, true, terms, "u");
                }
                for (int r = 0; r < d; ++r) {
                    if (t0) std::fprintf(f, "          const double g%d%s = t%db%s - t0b%s;\n", r, sj.c_str(), r + 1, sj.c_str(), sj.c_str());
                    else std::fprintf(f, "          const double g%d%s = t%db%s;\n", r, sj.c_str(), r + 1, sj.c_str());
                    flops += t0;
                }
                continue;
            }
            for (int b = 0; b < t.nblk; ++b) {
                std::vector<std::pair<int, Rat>> terms;
                for (int l = 0; l < VT; ++l)
                    if (!t.at(b, j, l).is_zero()) terms.push_back({l, t.at(b, j, l)});
                flops += emit_combo(f, "          ", "g" + std::to_string(b) + "_" + std::to_string(j), true, terms, "u");
            }
        }
        for (int j = j0; j < j1; ++j) {
            const std::string sj = "_" + std::to_string(j);
            if (form == 0) {
                std::fprintf(f, "          const double h0%s = pol.w(%d) * g0%s;\n", sj.c_str(), row(j), sj.c_str());
                flops += 1;
            } else if (store == 0) {
                for (int k = 0; k < NC; ++k)
                    std::fprintf(f, "          const double a%d%s = pol.w(%d);\n", k, sj.c_str(), row(j) + k);
                for (int r = 0; r < d; ++r) {
                    std::string acc = "a" + std::to_string(idx[r][0]) + sj + " * g0" + sj;
                    for (int s2 = 1; s2 < d; ++s2)
                        acc = "__fma_rn(a" + std::to_string(idx[r][s2]) + sj + ", g" + std::to_string(s2) + sj + ", " + acc + ")";
                    std::fprintf(f, "          const double h%d%s = %s;\n", r, sj.c_str(), acc.c_str());
                    flops += 2 * d - 1;
                }
            } else {
                std::fprintf(f, "          const double a%s = pol.w(%d);\n", sj.c_str(), row(j));
                for (int s2 = 0; s2 < d; ++s2)
                    std::fprintf(f, "          const double t%d%s = a%s * g%d%s;\n", s2, sj.c_str(), sj.c_str(), s2, sj.c_str());
                flops += d;
                for (int r = 0; r < d; ++r) {
                    std::string acc = "G" + std::to_string(idx[r][0]) + " * t0" + sj;
                    for (int s2 = 1; s2 < d; ++s2)
                        acc = "__fma_rn(G" + std::to_string(idx[r][s2]) + ", t" + std::to_string(s2) + sj + ", " + acc + ")";
                    std::fprintf(f, "          const double h%d%s = %s;\n", r, sj.c_str(), acc.c_str());
                    flops += 2 * d - 1;
                }
            }
            if (bary_p) {
                bool d0 = false;
                for (int l = 0; l < VT; ++l) d0 |= !D.at(0, j, l).is_zero();
                if (d0) {
                    std::string s = "h0" + sj;
                    for (int r = 1; r < d; ++r) s += " + h" + std::to_string(r) + sj;
                    std::fprintf(f, "          const double hs%s = %s;\n", sj.c_str(), s.c_str());
                    flops += d - 1;
                }
                for (int l = 0; l < VT; ++l) {
                    std::string acc = "y[" + std::to_string(l) + "]";
                    bool any = false;
                    for (int i = 0; i <= d; ++i) {
                        Rat cv = i == 0 ? Rat(0) - D.at(0, j, l) : D.at(i, j, l);
                        if (cv.is_zero()) continue;
                        any = true;
                        std::string h = i == 0 ? "hs" + sj : "h" + std::to_string(i - 1) + sj;
                        if (cv == Rat(1)) acc = "(" + acc + ") + " + h;
                        else if (cv == Rat(-1)) acc = "(" + acc + ") - " + h;
                        else { acc = "__fma_rn(" + lit(cv.to_double()) + ", " + h + ", " + acc + ")"; flops += 1; }
                        flops += 1;
                    }
                    if (any) std::fprintf(f, "          y[%d] = %s;\n", l, acc.c_str());
                }
                continue;
            }
            for (int l = 0; l < VT; ++l) {
                std::string acc = "y[" + std::to_string(l) + "]";
                bool any = false;
                for (int b = 0; b < t.nblk; ++b) {
                    Rat cv = t.at(b, j, l);
                    if (cv.is_zero()) continue;
                    any = true;
                    std::string h = "h" + std::to_string(b) + sj;
                    if (cv == Rat(1)) acc = "(" + acc + ") + " + h;
                    else if (cv == Rat(-1)) acc = "(" + acc + ") - " + h;
                    else { acc = "__fma_rn(" + lit(cv.to_double()) + ", " + h + ", " + acc + ")"; flops += 1; }
                    flops += 1;
                }
                if (any) std::fprintf(f, "          y[%d] = %s;\n", l, acc.c_str());
            }
        }
        for (int j = j0; j < j1; ++j) std::fprintf(f, "          pol.template end<%d>();\n", j);
        std::fprintf(f, "        }\n");
        j0 = j1;
    }
    std::fprintf(f, "    }\n");
    std::fprintf(f, "    static constexpr int FLOPS = %d;\n", flops);
    std::fprintf(f, "};\n\n");
}

// Symmetry-adapted WP variant (STORE 5).  G = an abelian group of commuting
// barycentric involutions (3D: <(0 1), (2 3)>, 2D: <(0 1)>).  Bhat is G-equivariant,
// Bhat[g beta, g alpha] = Bhat[beta, alpha] (product basis), so in
// symmetry-adapted coordinates -- per orbit O and character chi trivial on the
// stabiliser, uhat_chi(O) = sum_{g in G} chi(g) u_{g l0} -- it is block diagonal by
// character (Schur): ghat_chi(P) = sum_O Bhat_chi[P,O] uhat_chi(O),
// Bhat_chi[P,O] = sum_{l in O} chi(k_l) Bhat[j0(P), l].  The weights of an orbit P
// become the s x s matrix [ahat_{chi chi'}(P)], ahat_psi(P) = (1/|G|) sum_g psi(g) a_{g j0}
// (same count: s values per orbit, stored instead of a_j), and the projection uses
// Btilde_chi[P,O] = sum_{j in P} chi(k_j) Bhat[j, l0(O)].  3D P4: 784 block entries
// instead of 1729, ~2240 instead of ~3340 FP64 instructions per element.
// Emitted body: v = adapted u (butterflies), per W orbit: ghat (block rows), hhat =
// weight matrix x ghat, z += Btilde^T hhat; y = inverse butterflies of z / |G|.
// raw = true (STORE 6, internal): the plain element-wise weights a_{T,j} of
// DOGIP_STORE_FULL, rows permuted into the same orbit order (ROWPERM), and the body forms
// ahat_psi(P) = (1/s) sum_c psi(c) a_{c j0} from the orbit's s raw values (butterflies)
// before the weight multiply: FULL storage through the symmetry-adapted body.
static void emit_sym(FILE* f, int d, int p, bool raw = false) {
    Table t = bhat_table(d, p, 0);
    const int VT = t.cols, WT = t.rows;
    auto A = multi_indices(d, p);
    auto W = multi_indices(d, 2 * p);
    std::vector<std::array<int, 4>> gens;
    if (d == 3) gens = {{1, 0, 2, 3}, {0, 1, 3, 2}};
    else gens = {{1, 0, 2, 3}};
    const int ng = (int)gens.size(), NGR = 1 << ng;
    auto act = [&](const std::array<int, 4>& g, const std::array<int, 4>& a) {
        std::array<int, 4> b{};
        for (int i = 0; i <= d; ++i) b[i] = a[g[i]];
        return b;
    };
    auto compose = [&](const std::array<int, 4>& g, const std::array<int, 4>& h) {
        std::array<int, 4> r{};
        for (int i = 0; i < 4; ++i) r[i] = g[h[i]];
        return r;
    };
    // group element e (bitmask of generators) and character c (bitmask of -1 signs)
    std::vector<std::array<int, 4>> G(NGR);
    for (int e = 0; e < NGR; ++e) {
        std::array<int, 4> g{0, 1, 2, 3};
        for (int i = 0; i < ng; ++i)
            if (e >> i & 1) g = compose(g, gens[i]);
        G[e] = g;
    }
    auto chi = [&](int c, int e) { return (__builtin_popcount(c & e) & 1) ? -1 : 1; };
    auto find = [](const std::vector<std::array<int, 4>>& v, const std::array<int, 4>& a) {
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i] == a) return (int)i;
        std::fprintf(stderr, "sym: not found\n");
        std::exit(1);
    };
    std::vector<std::vector<int>> gV(NGR, std::vector<int>(VT)), gW(NGR, std::vector<int>(WT));
    for (int e = 0; e < NGR; ++e) {
        for (int l = 0; l < VT; ++l) gV[e][l] = find(A, act(G[e], A[l]));
        for (int j = 0; j < WT; ++j) gW[e][j] = find(W, act(G[e], W[j]));
    }
    for (int e = 0; e < NGR; ++e)
        for (int j = 0; j < WT; ++j)
            for (int l = 0; l < VT; ++l)
                if (t.at(0, gW[e][j], gV[e][l]) != t.at(0, j, l)) { std::fprintf(stderr, "sym: not equivariant\n"); std::exit(1); }
    struct Orb { int rep; std::vector<int> chars; std::vector<int> members; };   // chars trivial on the stabiliser
    auto orbits = [&](int n, const std::vector<std::vector<int>>& gx) {
        std::vector<Orb> out;
        std::vector<bool> seen(n, false);
        for (int i = 0; i < n; ++i) {
            if (seen[i]) continue;
            Orb o; o.rep = i;
            for (int e = 0; e < NGR; ++e) {
                const int k = gx[e][i];
                if (!seen[k]) { seen[k] = true; o.members.push_back(k); }
            }
            for (int c = 0; c < NGR; ++c) {
                bool triv = true;
                for (int e = 0; e < NGR; ++e)
                    if (gx[e][i] == i && chi(c, e) != 1) triv = false;
                if (triv) o.chars.push_back(c);
            }
            out.push_back(o);
        }
        return out;
    };
    auto OV = orbits(VT, gV), OW0 = orbits(WT, gW);
    // W orbits by decreasing size: weight rows of an orbit never straddle a chunk of 4k rows
    std::vector<Orb> OW;
    for (int sz = NGR; sz >= 1; sz /= 2)
        for (auto& o : OW0)
            if ((int)o.members.size() == sz) OW.push_back(o);
    // adapted V index of (orbit, char)
    std::vector<std::vector<int>> vidx(OV.size());
    int nv = 0;
    for (size_t o = 0; o < OV.size(); ++o)
        for (size_t c = 0; c < OV[o].chars.size(); ++c) vidx[o].push_back(nv++);
    // weight rows (orbit P, char psi) and the weights-kernel recombination table
    std::vector<std::vector<int>> wrow(OW.size());
    std::vector<std::array<int, 4>> rj;
    std::vector<std::array<Rat, 4>> rc;
    int nr = 0;
    for (size_t P = 0; P < OW.size(); ++P) {
        const int s = (int)OW[P].members.size();
        for (int psi : OW[P].chars) {
            wrow[P].push_back(nr++);
            // ahat_psi = (1/|G|) sum_g psi(g) a_{g j0} = (1/s) sum over distinct members
            std::array<int, 4> js{-1, -1, -1, -1};
            std::array<Rat, 4> cs{};
            int k = 0;
            for (int e = 0; e < NGR; ++e) {
                const int j = gW[e][OW[P].rep];
                bool dup = false;
                for (int q = 0; q < k; ++q)
                    if (js[q] == j) dup = true;
                if (dup) continue;
                js[k] = j;
                cs[k] = Rat(chi(psi, e), s);
                ++k;
            }
            rj.push_back(js);
            rc.push_back(cs);
        }
    }
    int nnz = 0, pm1 = 0;
    for (auto& v : t.v) { nnz += !v.is_zero(); pm1 += v.is_pm1(); }
    auto simp = cell_simplices(d);
    std::fprintf(f, "template <> struct RefElem<%d, %d, 0, %d> {\n", d, p, raw ? 6 : 5);
    std::fprintf(f, "    static constexpr int VT = %d, WT = %d, NC = 1, NG = 0, ROWS = 12, TILE_ROWS = %d, NS = %d, RALIGN = %d, PAIR = 0, DOT_IN_BODY = 1, HAS_ROWPERM = %d;\n",
                 VT, WT, WT, (int)simp.size(), NGR, raw ? 1 : 0);
    std::fprintf(f, "    static constexpr int NNZ = %d, NNZ_PM1 = %d, NGROUP = %d;\n", nnz, pm1, NGR);
    std::fprintf(f, "    static constexpr signed char LOFF[%d][%d][%d] = {", (int)simp.size(), VT, d);
    for (size_t si = 0; si < simp.size(); ++si) {
        std::fprintf(f, "%s{", si ? ", " : "");
        for (int l = 0; l < VT; ++l) {
            std::fprintf(f, "%s{", l ? "," : "");
            for (int ax = 0; ax < d; ++ax) {
                int o = 0;
                for (int i = 0; i <= d; ++i) o += A[l][i] * simp[si][i][ax];
                std::fprintf(f, "%s%d", ax ? "," : "", o);
            }
            std::fprintf(f, "}");
        }
        std::fprintf(f, "}");
    }
    std::fprintf(f, "};\n");
    std::fprintf(f, "    static constexpr signed char ALPHA[%d][3] = {", VT);
    for (int l = 0; l < VT; ++l)
        std::fprintf(f, "%s{%d,%d,%d}", l ? "," : "", A[l][1], A[l][2], d == 3 ? A[l][3] : 0);
    std::fprintf(f, "};\n");
    if (raw) {
        // ROWPERM[j] = stored row of W node j: member k of orbit P (in the order of rj) at
        // row wrow[P][0] + k
        std::vector<int> perm(WT, -1);
        for (size_t P = 0; P < OW.size(); ++P)
            for (int k = 0; k < 4; ++k) {
                const int j = rj[wrow[P][0]][k];
                if (j >= 0) perm[j] = wrow[P][0] + k;
            }
        std::fprintf(f, "    static constexpr short ROWPERM[%d] = {", WT);
        for (int j = 0; j < WT; ++j) {
            if (perm[j] < 0) { std::fprintf(stderr, "sym raw: node without a row\n"); std::exit(1); }
            std::fprintf(f, "%s%d", j ? "," : "", perm[j]);
        }
        std::fprintf(f, "};\n");
    }
    // weights-kernel table: stored row r = sum_k SYMC[r][k] a_{SYMJ[r][k]}
    if (!raw) {
    std::fprintf(f, "    static constexpr short SYMJ[%d][4] = {", WT);
    for (int r = 0; r < WT; ++r)
        std::fprintf(f, "%s{%d,%d,%d,%d}", r ? "," : "", rj[r][0], rj[r][1], rj[r][2], rj[r][3]);
    std::fprintf(f, "};\n");
    std::fprintf(f, "    static constexpr double SYMC[%d][4] = {", WT);
    for (int r = 0; r < WT; ++r)
        std::fprintf(f, "%s{%s,%s,%s,%s}", r ? "," : "", lit(rc[r][0].to_double()).c_str(), lit(rc[r][1].to_double()).c_str(),
                     lit(rc[r][2].to_double()).c_str(), lit(rc[r][3].to_double()).c_str());
    std::fprintf(f, "};\n");
    }
    std::fprintf(f, "    static __host__ __device__ constexpr int row_of(int r) { return r; }\n");
    // dot != null: *dot += u_T . y_T, computed as v . z (Parseval over the characters:
    // sum_k v_k z_k = sum_l u_l y_l), so u_T dies after the transform (issuing the next
    // tile's gather there instead measured slower: it keeps 35 more doubles live)
    std::fprintf(f,
        "    template <class Pol>\n"
        "    static __device__ __forceinline__ void body(const double* __restrict__ u,\n"
        "                                                double* __restrict__ y, Pol& pol, double* dot) {\n");
    int flops = 0;
    // 1. adapted coordinates v[k] = sum_{cosets} chi(c) u_{c l0} (stabiliser multiplicity
    //    folded into the block constants): butterflies over the generators
    std::fprintf(f, "        DOGIP_SYM_VDECL(%d);\n        double z[%d];\n", VT, VT);
    // v index -> u_T slot of the same orbit (read-all-then-write per orbit, so v can
    // overwrite u in place when it lives in the shared-memory staging buffer)
    static std::vector<int> vslot;
    vslot.assign(VT, -1);
    auto coset_sum = [&](const Orb& o, int c, int gen_bits, const std::vector<std::vector<int>>& gx) {
        // distinct members with their sign: sum over e of chi(c,e) x_{e rep}, distinct only
        std::vector<std::pair<int, int>> terms;
        for (int e = 0; e < NGR; ++e) {
            const int k = gx[e][o.rep];
            bool dup = false;
            for (auto& tm : terms)
                if (tm.first == k) dup = true;
            if (!dup) terms.push_back({k, chi(c, e)});
        }
        (void)gen_bits;
        return terms;
    };
    for (size_t o = 0; o < OV.size(); ++o) {
        const Orb& O = OV[o];
        const int sz = (int)O.members.size();
        if (sz == 1) {
            vslot[vidx[o][0]] = O.rep;
            std::fprintf(f, "        DOGIP_SYM_VSET(%d, %d, DOGIP_SYM_U(%d));\n", vidx[o][0], O.rep, O.rep);
            continue;
        }
        if (sz == 2) {
            auto tm = coset_sum(O, 0, 0, gV);
            const int a = tm[0].first, b = tm[1].first;
            vslot[vidx[o][0]] = a;
            vslot[vidx[o][1]] = b;
            std::fprintf(f, "        { const double ua = DOGIP_SYM_U(%d), ub = DOGIP_SYM_U(%d);\n", a, b);
            std::fprintf(f, "          DOGIP_SYM_VSET(%d, %d, ua + ub);\n", vidx[o][0], a);
            std::fprintf(f, "          DOGIP_SYM_VSET(%d, %d, ua - ub);\n        }\n", vidx[o][1], b);
            flops += 2;
            continue;
        }
        // size 4: members a = e0, b = g1 a, c = g2 a, d = g1 g2 a; chars (s1, s2)
        const int a = gV[0][O.rep], b = gV[1][O.rep], c = gV[2][O.rep], dd = gV[3][O.rep];
        const int mem[4] = {a, b, c, dd};
        std::fprintf(f, "        { const double ua = DOGIP_SYM_U(%d), ub = DOGIP_SYM_U(%d), uc = DOGIP_SYM_U(%d), ud = DOGIP_SYM_U(%d);\n",
                     a, b, c, dd);
        std::fprintf(f, "          const double tp = ua + ub, tm = ua - ub, rp = uc + ud, rm = uc - ud;\n");
        for (size_t ci = 0; ci < O.chars.size(); ++ci) {
            const int ch = O.chars[ci];
            const bool s1 = ch & 1, s2 = ch & 2;   // chi(g1) = -1 if bit 0, chi(g2) = -1 if bit 1
            vslot[vidx[o][ci]] = mem[ci];
            std::fprintf(f, "          DOGIP_SYM_VSET(%d, %d, %s %s %s);\n", vidx[o][ci], mem[ci], s1 ? "tm" : "tp", s2 ? "-" : "+", s1 ? "rm" : "rp");
        }
        std::fprintf(f, "        }\n");
        flops += 8;
    }
    std::fprintf(f, "#pragma unroll\n        for (int k = 0; k < %d; ++k) z[k] = 0.0;\n", VT);
    // 2-4. per W orbit
    for (size_t P = 0; P < OW.size(); ++P) {
        const Orb& PO = OW[P];
        const int j0 = PO.rep;
        std::fprintf(f, "        {\n          pol.template begin<%d>();\n", wrow[P][0]);
        // the orbit's weights first: their shared-memory latency overlaps the block rows
        if (!raw) {
            for (size_t q = 0; q < PO.chars.size(); ++q)
                std::fprintf(f, "          const double a%zu = pol.w(%d);\n", q, wrow[P][q]);
        } else {
            // raw a_{member k} at row wrow[P][0] + k; ahat_q = sum_k rc[q][k] r_k, rc = +-1/s
            const int s = (int)PO.members.size();
            for (int k = 0; k < s; ++k) std::fprintf(f, "          const double r%d = pol.w(%d);\n", k, wrow[P][0] + k);
            auto sgn = [&](int q, int k) { return rc[wrow[P][q]][k].to_double() > 0 ? 1 : -1; };
            if (s == 1) {
                std::fprintf(f, "          const double a0 = r0;\n");
            } else if (s == 2) {
                for (int q = 0; q < 2; ++q)
                    std::fprintf(f, "          const double a%d = (r0 %s r1) * 0.5;\n", q, sgn(q, 1) > 0 ? "+" : "-");
                flops += 4;
            } else {
                // members k = 0..3 are e = 0..3 (distinct): ahat = ((r0 + s1 r1) + s2 (r2 + s1 r3)) / 4
                for (int k = 0; k < 4; ++k)
                    if (rj[wrow[P][0]][k] != gW[k][j0]) { std::fprintf(stderr, "sym raw: member order\n"); std::exit(1); }
                std::fprintf(f, "          const double tp = r0 + r1, tm = r0 - r1, rp = r2 + r3, rm = r2 - r3;\n");
                for (int q = 0; q < 4; ++q) {
                    const bool s1 = sgn(q, 1) < 0, s2 = sgn(q, 2) < 0;
                    if (sgn(q, 3) != (s1 == s2 ? 1 : -1)) { std::fprintf(stderr, "sym raw: character\n"); std::exit(1); }
                    std::fprintf(f, "          const double a%d = (%s %s %s) * 0.25;\n", q, s1 ? "tm" : "tp", s2 ? "-" : "+", s1 ? "rm" : "rp");
                }
                flops += 12;
            }
        }
        // ghat_chi = sum_O Bhat_chi[P,O] uhat_chi(O), uhat = |H_O| v
        for (size_t ci = 0; ci < PO.chars.size(); ++ci) {
            const int ch = PO.chars[ci];
            std::vector<std::pair<int, Rat>> terms;
            for (size_t o = 0; o < OV.size(); ++o) {
                const Orb& O = OV[o];
                int cpos = -1;
                for (size_t q = 0; q < O.chars.size(); ++q)
                    if (O.chars[q] == ch) cpos = (int)q;
                if (cpos < 0) continue;
                Rat sum(0);
                for (int e = 0; e < NGR; ++e) sum = sum + Rat(chi(ch, e)) * t.at(0, j0, gV[e][O.rep]);
                // sum over the full group = |H_O| * sum over distinct members; uhat = |H_O| v
                // -> ghat = sum_O (sum_{l in O} chi B[j0,l]) |H_O| v = sum_O sum_g chi(g) B[j0, g l0] v
                if (!sum.is_zero()) terms.push_back({vidx[o][cpos], sum});
            }
            g_vslot = &vslot;
            flops += emit_combo(f, "          ", "g" + std::to_string(ci), true, terms, "V");
            g_vslot = nullptr;
        }
        // hhat_chi = sum_chi' ahat_{chi chi'} ghat_chi'  (ahat rows of this orbit)
        for (size_t ci = 0; ci < PO.chars.size(); ++ci) {
            std::string acc;
            for (size_t cj = 0; cj < PO.chars.size(); ++cj) {
                const int psi = PO.chars[ci] ^ PO.chars[cj];
                int rpos = -1;
                for (size_t q = 0; q < PO.chars.size(); ++q)
                    if (PO.chars[q] == psi) rpos = (int)q;
                const std::string w = "a" + std::to_string(rpos);
                const std::string gj = "g" + std::to_string(cj);
                if (acc.empty()) { acc = w + " * " + gj; flops += 1; }
                else { acc = "__fma_rn(" + w + ", " + gj + ", " + acc + ")"; flops += 2; }
            }
            std::fprintf(f, "          const double h%zu = %s;\n", ci, acc.c_str());
        }
        // z_chi(O) += Btilde_chi[P,O] hhat_chi(P) / |G|,  Btilde = sum_{j in P} chi(k_j) B[j, l0(O)]
        for (size_t o = 0; o < OV.size(); ++o) {
            const Orb& O = OV[o];
            for (size_t q = 0; q < O.chars.size(); ++q) {
                const int ch = O.chars[q];
                int cpos = -1;
                for (size_t ci = 0; ci < PO.chars.size(); ++ci)
                    if (PO.chars[ci] == ch) cpos = (int)ci;
                if (cpos < 0) continue;
                Rat sum(0);
                std::vector<int> seen;
                for (int e = 0; e < NGR; ++e) {
                    const int j = gW[e][j0];
                    bool dup = false;
                    for (int x : seen) if (x == j) dup = true;
                    if (dup) continue;
                    seen.push_back(j);
                    sum = sum + Rat(chi(ch, e)) * t.at(0, j, O.rep);
                }
                sum = sum * Rat(1, NGR);
                if (sum.is_zero()) continue;
                const int k = vidx[o][q];
                const std::string h = "h" + std::to_string(cpos);
                std::string acc = "z[" + std::to_string(k) + "]";
                if (sum == Rat(1)) acc = "(" + acc + ") + " + h;
                else if (sum == Rat(-1)) acc = "(" + acc + ") - " + h;
                else { acc = "__fma_rn(" + lit(sum.to_double()) + ", " + h + ", " + acc + ")"; flops += 1; }
                flops += 1;
                std::fprintf(f, "          z[%d] = %s;\n", k, acc.c_str());
            }
        }
        std::fprintf(f, "        }\n");
    }
    // 5. y_{c l0} = sum_chi chi(c) z_chi (the 1/|G| is in the projection constants)
    for (size_t o = 0; o < OV.size(); ++o) {
        const Orb& O = OV[o];
        const int sz = (int)O.members.size();
        if (sz == 1) {
            std::fprintf(f, "        y[%d] += z[%d];\n", O.rep, vidx[o][0]);
            flops += 1;
            continue;
        }
        // member e-rep gets sum_chi chi(e) z_chi
        std::vector<int> done;
        for (int e = 0; e < NGR; ++e) {
            const int m = gV[e][O.rep];
            bool dup = false;
            for (int x : done) if (x == m) dup = true;
            if (dup) continue;
            done.push_back(m);
            std::string acc;
            for (size_t q = 0; q < O.chars.size(); ++q) {
                const std::string zz = "z[" + std::to_string(vidx[o][q]) + "]";
                if (acc.empty()) acc = chi(O.chars[q], e) > 0 ? zz : "-" + zz;
                else acc = "(" + acc + (chi(O.chars[q], e) > 0 ? ") + " : ") - ") + zz;
            }
            std::fprintf(f, "        y[%d] += %s;\n", m, acc.c_str());
            flops += (int)O.chars.size();
        }
    }
    std::fprintf(f, "        if (dot) {\n          double s = 0.0;\n");
    for (int k = 0; k < VT; ++k) std::fprintf(f, "          s = fma(DOGIP_SYM_V(%d, %d), z[%d], s);\n", k, vslot[k], k);
    std::fprintf(f, "          *dot += s;\n        }\n");
    std::fprintf(f, "    }\n");
    std::fprintf(f, "    static constexpr int FLOPS = %d;\n", flops);
    std::fprintf(f, "};\n\n");
}

// Symmetry-adapted body of the isotropic EL storage (STORE 1, corollary P:411-428):
// sigma = (1 2) swaps xhat_1 <-> xhat_2, i.e. the gradient components r = 0 <-> 1, and
// Bhat_EL is equivariant, Bhat[s r][sigma j][sigma l] = Bhat[r][j][l].  With
// v+ = u_l + u_{sigma l}, v- = u_l - u_{sigma l} (DoF pairs) the gradients of a node pair
// (j, jj = sigma j) are g_r(j) = P_r + Q_r, g_{s r}(jj) = P_r - Q_r with P_r from the
// even and Q_r from the odd half of row (r, j) -- each half has ~1/3 fewer nonzeros
// (3D P3: 690 instead of 1014).  The weights act in the original basis (h = a_j G g),
// then H+/-_r = h_r(j) +/- h_{s r}(jj) feed the transposed halves; y_l, y_{sigma l} are
// recovered from the even / odd accumulators.  Node pairs are stored in adjacent rows.
static void emit_iso_sym(FILE* f, int d, int p) {
    Table t = bhat_table(d, p, 1);
    const int VT = t.cols, WT = t.rows;
    const int NSYM = d * (d + 1) / 2, NG = NSYM;
    auto A = multi_indices(d, p);
    auto W = multi_indices(d, 2 * p - 2);
    const int sig[4] = {0, 2, 1, 3};       // barycentric lambda_1 <-> lambda_2
    const int sr[3] = {1, 0, 2};           // gradient components
    auto perm = [&](const std::array<int, 4>& a) {
        std::array<int, 4> b{};
        for (int i = 0; i <= d; ++i) b[i] = a[sig[i]];
        return b;
    };
    auto find = [](const std::vector<std::array<int, 4>>& v, const std::array<int, 4>& a) {
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i] == a) return (int)i;
        std::fprintf(stderr, "iso-sym: not found\n");
        std::exit(1);
    };
    std::vector<int> sA(VT), sW(WT);
    for (int l = 0; l < VT; ++l) sA[l] = find(A, perm(A[l]));
    for (int j = 0; j < WT; ++j) sW[j] = find(W, perm(W[j]));
    for (int r = 0; r < d; ++r)
        for (int j = 0; j < WT; ++j)
            for (int l = 0; l < VT; ++l)
                if (t.at(sr[r], sW[j], sA[l]) != t.at(r, j, l)) { std::fprintf(stderr, "iso-sym: not equivariant\n"); std::exit(1); }
    std::vector<std::pair<int, int>> vp;   // DoF pairs (l < sigma l)
    std::vector<int> vf;                   // fixed DoFs
    for (int l = 0; l < VT; ++l) {
        if (sA[l] > l) vp.push_back({l, sA[l]});
        else if (sA[l] == l) vf.push_back(l);
    }
    std::vector<std::pair<int, int>> wp;   // node pairs
    std::vector<int> wf;
    for (int j = 0; j < WT; ++j) {
        if (sW[j] > j) wp.push_back({j, sW[j]});
        else if (sW[j] == j) wf.push_back(j);
    }
    // storage rows: G (NG rows), then node pairs adjacent, then fixed nodes
    std::vector<int> rowperm(WT);
    int nr = 0;
    for (auto& pr : wp) { rowperm[pr.first] = nr++; rowperm[pr.second] = nr++; }
    for (int j : wf) rowperm[j] = nr++;
    // adapted coordinates: vs[i], vd[i] for pair i; u[vf] directly
    const int NP = (int)vp.size(), NF = (int)vf.size();
    int nnz = 0, pm1 = 0;
    for (auto& v : t.v) { nnz += !v.is_zero(); pm1 += v.is_pm1(); }
    auto simp = cell_simplices(d);
    std::fprintf(f, "template <> struct RefElem<%d, %d, 1, 1> {\n", d, p);
    std::fprintf(f, "    static constexpr int VT = %d, WT = %d, NC = 1, NG = %d, ROWS = 12, TILE_ROWS = %d, NS = %d, RALIGN = 1, PAIR = 0, DOT_IN_BODY = 0, HAS_ROWPERM = 1;\n",
                 VT, WT, NG, NG + WT, (int)simp.size());
    std::fprintf(f, "    static constexpr int NNZ = %d, NNZ_PM1 = %d;\n", nnz, pm1);
    std::fprintf(f, "    static constexpr signed char LOFF[%d][%d][%d] = {", (int)simp.size(), VT, d);
    for (size_t si = 0; si < simp.size(); ++si) {
        std::fprintf(f, "%s{", si ? ", " : "");
        for (int l = 0; l < VT; ++l) {
            std::fprintf(f, "%s{", l ? "," : "");
            for (int ax = 0; ax < d; ++ax) {
                int o = 0;
                for (int i = 0; i <= d; ++i) o += A[l][i] * simp[si][i][ax];
                std::fprintf(f, "%s%d", ax ? "," : "", o);
            }
            std::fprintf(f, "}");
        }
        std::fprintf(f, "}");
    }
    std::fprintf(f, "};\n");
    std::fprintf(f, "    static constexpr signed char ALPHA[%d][3] = {", VT);
    for (int l = 0; l < VT; ++l)
        std::fprintf(f, "%s{%d,%d,%d}", l ? "," : "", A[l][1], A[l][2], d == 3 ? A[l][3] : 0);
    std::fprintf(f, "};\n");
    std::fprintf(f, "    static constexpr short ROWPERM[%d] = {", WT);
    for (int j = 0; j < WT; ++j) std::fprintf(f, "%s%d", j ? "," : "", rowperm[j]);
    std::fprintf(f, "};\n");
    std::fprintf(f, "    static __host__ __device__ constexpr int row_of(int r) { return r; }\n");
    std::fprintf(f,
        "    template <class Pol>\n"
        "    static __device__ __forceinline__ void body(const double* __restrict__ u,\n"
        "                                                double* __restrict__ y, Pol& pol) {\n");
    int flops = 0;
    int idx[3][3], c = 0;
    for (int r = 0; r < d; ++r)
        for (int s2 = r; s2 < d; ++s2) { idx[r][s2] = idx[s2][r] = c++; }
    // inputs: v[0..NP) = u_l + u_sl, v[NP..2NP) = u_l - u_sl, v[2NP + k] = u_{vf[k]}
    std::fprintf(f, "        double v[%d], zs[%d], zd[%d], zf[%d];\n", VT, NP > 0 ? NP : 1, NP > 0 ? NP : 1, NF > 0 ? NF : 1);
    for (int i = 0; i < NP; ++i) {
        std::fprintf(f, "        v[%d] = u[%d] + u[%d];\n        v[%d] = u[%d] - u[%d];\n", i, vp[i].first, vp[i].second,
                     NP + i, vp[i].first, vp[i].second);
        flops += 2;
    }
    for (int k = 0; k < NF; ++k) std::fprintf(f, "        v[%d] = u[%d];\n", 2 * NP + k, vf[k]);
    std::fprintf(f, "#pragma unroll\n        for (int k = 0; k < %d; ++k) { zs[k] = 0.0; zd[k] = 0.0; }\n", NP > 0 ? NP : 1);
    std::fprintf(f, "#pragma unroll\n        for (int k = 0; k < %d; ++k) zf[k] = 0.0;\n", NF > 0 ? NF : 1);
    std::fprintf(f, "        pol.template begin<0>();\n");
    for (int k = 0; k < NSYM; ++k) std::fprintf(f, "        const double G%d = pol.w(%d);\n", k, k);
    // row (r, j) in adapted inputs: even part over vs (+ fixed DoFs), odd part over vd
    auto even_terms = [&](int r, int j) {
        std::vector<std::pair<int, Rat>> terms;
        for (int i = 0; i < NP; ++i) {
            const Rat cc = (t.at(r, j, vp[i].first) + t.at(r, j, vp[i].second)) * Rat(1, 2);
            if (!cc.is_zero()) terms.push_back({i, cc});
        }
        for (int k = 0; k < NF; ++k)
            if (!t.at(r, j, vf[k]).is_zero()) terms.push_back({2 * NP + k, t.at(r, j, vf[k])});
        return terms;
    };
    auto odd_terms = [&](int r, int j) {
        std::vector<std::pair<int, Rat>> terms;
        for (int i = 0; i < NP; ++i) {
            const Rat cc = (t.at(r, j, vp[i].first) - t.at(r, j, vp[i].second)) * Rat(1, 2);
            if (!cc.is_zero()) terms.push_back({NP + i, cc});
        }
        return terms;
    };
    auto weights = [&](const std::string& a, const std::string& g, const std::string& h) {
        // h = a * G * g (G symmetric, upper triangle G0..)
        for (int s2 = 0; s2 < d; ++s2) std::fprintf(f, "          const double t%s%d = %s * %s%d;\n", h.c_str(), s2, a.c_str(), g.c_str(), s2);
        flops += d;
        for (int r = 0; r < d; ++r) {
            std::string acc = "G" + std::to_string(idx[r][0]) + " * t" + h + "0";
            for (int s2 = 1; s2 < d; ++s2)
                acc = "__fma_rn(G" + std::to_string(idx[r][s2]) + ", t" + h + std::to_string(s2) + ", " + acc + ")";
            std::fprintf(f, "          const double %s%d = %s;\n", h.c_str(), r, acc.c_str());
            flops += 2 * d - 1;
        }
    };
    // projection of original-basis contributions (r, j, value) into zs / zd / zf
    auto project_even = [&](int r, int j, const std::string& val) {
        for (int i = 0; i < NP; ++i) {
            const Rat cc = (t.at(r, j, vp[i].first) + t.at(r, j, vp[i].second)) * Rat(1, 2);
            if (cc.is_zero()) continue;
            std::fprintf(f, "          zs[%d] = __fma_rn(%s, %s, zs[%d]);\n", i, lit(cc.to_double()).c_str(), val.c_str(), i);
            flops += 2;
        }
        for (int k = 0; k < NF; ++k) {
            const Rat cc = t.at(r, j, vf[k]);
            if (cc.is_zero()) continue;
            std::fprintf(f, "          zf[%d] = __fma_rn(%s, %s, zf[%d]);\n", k, lit(cc.to_double()).c_str(), val.c_str(), k);
            flops += 2;
        }
    };
    auto project_odd = [&](int r, int j, const std::string& val) {
        for (int i = 0; i < NP; ++i) {
            const Rat cc = (t.at(r, j, vp[i].first) - t.at(r, j, vp[i].second)) * Rat(1, 2);
            if (cc.is_zero()) continue;
            std::fprintf(f, "          zd[%d] = __fma_rn(%s, %s, zd[%d]);\n", i, lit(cc.to_double()).c_str(), val.c_str(), i);
            flops += 2;
        }
    };
    for (size_t q = 0; q < wp.size(); ++q) {
        const int j = wp[q].first, jj = wp[q].second;
        const int r0 = NG + rowperm[j];
        // both rows opened in order: with an odd NG (2D) a pair can straddle two chunks;
        // aj is read before the second begin may move to the next stage
        std::fprintf(f, "        {\n          pol.template begin<%d>();\n", r0);
        std::fprintf(f, "          const double aj = pol.w(%d);\n", r0);
        std::fprintf(f, "          pol.template begin<%d>();\n", r0 + 1);
        std::fprintf(f, "          const double ajj = pol.w(%d);\n", r0 + 1);
        for (int r = 0; r < d; ++r) {
            flops += emit_combo(f, "          ", "P" + std::to_string(r), true, even_terms(r, j), "v");
            flops += emit_combo(f, "          ", "Q" + std::to_string(r), true, odd_terms(r, j), "v");
        }
        // g(j)_r = P_r + Q_r ; g(jj)_s = P_{sr s} - Q_{sr s}
        for (int r = 0; r < d; ++r) std::fprintf(f, "          const double ga%d = P%d + Q%d;\n", r, r, r);
        for (int s2 = 0; s2 < d; ++s2) std::fprintf(f, "          const double gb%d = P%d - Q%d;\n", s2, sr[s2], sr[s2]);
        flops += 2 * d;
        weights("aj", "ga", "ha");
        weights("ajj", "gb", "hb");
        // H+_r = ha_r + hb_{sr r}, H-_r = ha_r - hb_{sr r}
        for (int r = 0; r < d; ++r) {
            std::fprintf(f, "          const double Hp%d = ha%d + hb%d, Hm%d = ha%d - hb%d;\n", r, r, sr[r], r, r, sr[r]);
            flops += 2;
        }
        // pair contribution: y_l + y_sl = sum_r (B_l + B_sl) H+_r (even, fixed DoFs: B_f H+_r),
        //                    y_l - y_sl = sum_r (B_l - B_sl) H-_r
        for (int r = 0; r < d; ++r) project_even(r, j, "Hp" + std::to_string(r));
        for (int r = 0; r < d; ++r) project_odd(r, j, "Hm" + std::to_string(r));
        std::fprintf(f, "        }\n");
    }
    for (int j : wf) {
        const int r0 = NG + rowperm[j];
        std::fprintf(f, "        {\n          pol.template begin<%d>();\n", r0);
        std::fprintf(f, "          const double aj = pol.w(%d);\n", r0);
        for (int r = 0; r < d; ++r) {
            flops += emit_combo(f, "          ", "P" + std::to_string(r), true, even_terms(r, j), "v");
            flops += emit_combo(f, "          ", "Q" + std::to_string(r), true, odd_terms(r, j), "v");
            std::fprintf(f, "          const double ga%d = P%d + Q%d;\n", r, r, r);
            flops += 1;
        }
        weights("aj", "ga", "ha");
        // original-basis projection of h(j): y_l = sum_r B_l h_r, y_sl = sum_r B_sl h_r
        for (int r = 0; r < d; ++r) {
            project_even(r, j, "ha" + std::to_string(r));
            project_odd(r, j, "ha" + std::to_string(r));
        }
        std::fprintf(f, "        }\n");
    }
    // y_l = zs + zd, y_sl = zs - zd, y_f = zf  (the 1/2 of the averages is in the constants:
    // zs = (y_l + y_sl)/2, zd = (y_l - y_sl)/2)
    for (int i = 0; i < NP; ++i) {
        std::fprintf(f, "        y[%d] += zs[%d] + zd[%d];\n        y[%d] += zs[%d] - zd[%d];\n", vp[i].first, i, i,
                     vp[i].second, i, i);
        flops += 4;
    }
    for (int k = 0; k < NF; ++k) { std::fprintf(f, "        y[%d] += zf[%d];\n", vf[k], k); flops += 1; }
    std::fprintf(f, "    }\n");
    std::fprintf(f, "    static constexpr int FLOPS = %d;\n", flops);
    std::fprintf(f, "};\n\n");
}

static int g_iso_sym = 0;   // argv[5]: 1 = symmetry-adapted ISO body (measured slower: spills, see DESIGN)

int main(int argc, char** argv) {
    if (argc < 2) { std::fprintf(stderr, "usage: gen_bhat out.cuh [group_values]\n"); return 2; }
    if (argc > 2) g_gmax_vals = std::atoi(argv[2]);
    if (argc > 3) g_split = std::atoi(argv[3]);
    if (argc > 5) g_iso_sym = std::atoi(argv[5]);
    if (argc > 6) g_bary = std::atoi(argv[6]);
    FILE* f = std::fopen(argv[1], "w");
    if (!f) { std::perror("open"); return 1; }
    std::fprintf(f,
        "// AUTO-GENERATED by csrc/gen/gen_bhat.cpp from the exact tables of host/tables.hpp.\n"
        "// Do not edit.  One specialisation RefElem<D,P,FORM,STORE> per (d, p, form, storage):\n"
        "//   VT = C(p+d,d), WT = #double-grid nodes, NC = streamed rows per node,\n"
        "//   NG = leading per-element rows (iso storage: G_T = Rinv Rinv^T upper triangle),\n"
        "//   ROWS = rows per streamed chunk, TILE_ROWS = NG + WT*NC rows per 32-element tile,\n"
        "//   FLOPS = fp64 flops of body() per element (sparse, +-1 aware),\n"
        "//   NNZ / NNZ_PM1 = nnz Bhat / nnz_{+-1} Bhat (eq:comp_eff, PAPER.md P:548),\n"
        "//   LOFF[s][l][a] = DoF-lattice offset (axis a) of local DoF l of simplex s\n"
        "//                   inside its cell, in units of the DoF lattice.\n"
        "#pragma once\n\n"
        "// v of the symmetry-adapted bodies: registers unless the includer defines these\n"
        "#ifndef DOGIP_SYM_VDECL\n"
        "#define DOGIP_SYM_VDECL(n) double v[n]\n"
        "#define DOGIP_SYM_VSET(k, slot, e) (v[k] = (e))\n"
        "#define DOGIP_SYM_V(k, slot) v[k]\n"
        "#define DOGIP_SYM_U(l) u[l]\n"
        "#endif\n\n"
        "namespace dogip_gen {\n\n"
        "template <int D, int P, int FORM, int STORE> struct RefElem;\n\n");
    for (int d = 2; d <= 3; ++d)
        for (int p = 1; p <= 4; ++p) {
            emit_variant(f, d, p, 0, 0);
            emit_variant(f, d, p, 1, 0);
            if (g_iso_sym) emit_iso_sym(f, d, p);
            else emit_variant(f, d, p, 1, 1);
            emit_sym(f, d, p);
            emit_sym(f, d, p, true);
        }
    std::fprintf(f, "}  // namespace dogip_gen\n");
    std::fclose(f);
    return 0;
}
