// MIDBF factorization on the host with batched entry sampling, and the
// drop-in apply that forwards to the device plan.
//
// Follows reference src/butterfly.cpp:
//   idbf_factorize :708-769, shared_sweep :413-622, split_side :380-408,
//   sample_ids :360-369, leaf_side :279-293, check_inputs :295-305,
//   stream derivation :18-27.
// The one structural change is batching: the reference evaluates K inside
// each (system, unit) OpenMP task; here every sweep pass first gathers all of
// its (row ids x column ids) blocks and fills them in ONE call of a `Filler`
// (the GPU sampler K3 for a KernelDesc, or a host EntryFn loop), then runs the
// IDs on the host under OpenMP.  Draw order, stream seeds, block placement and
// grouping are the reference's, so a host-filled factorization is identical to
// the reference algorithm's.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <utility>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../device/sample.hpp"
#include "../status.hpp"
#include "midbf/butterfly.hpp"
#include "midbf_internal.hpp"

namespace midbf::bf {
namespace {

std::uint64_t mix(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// A contiguous run of ids owned by one tree node at the current unit level;
// `begin` is its offset inside its side.
struct Cell {
  Index node = 0;
  Index begin = 0;
  IndexVec ids;
};
struct Span {  // one side of a system
  int level = 0;
  std::vector<Cell> cells;
  Index size = 0;
  Index off = 0;
};
struct System {
  Span row, col;
};
struct Skel {  // interpolation operator + kept global ids of one cell
  MatXc M;
  IndexVec keep;
};

struct FillJob {
  const Index* rows;
  Index nr;
  const Index* cols;
  Index nc;
  MatXc* out;
};
using Filler = std::function<void(std::vector<FillJob>&)>;

// One interpolative decomposition of K(rows, cols): a row ID (W: nr x k,
// skeleton rows) or a column ID (V: k x nc, skeleton columns).
struct IdJob {
  const Index* rows;
  Index nr;
  const Index* cols;
  Index nc;
};
struct IdRes {
  MatXc M;
  IndexVec pos;
};
using IdFn = std::function<void(const std::vector<IdJob>&, bool rowid, std::vector<IdRes>&)>;

// Host IDs (src/butterfly.cpp:466-472, 516-519): fill the blocks, then
// la::rid_from_cols / la::cid_from_rows under OpenMP.
void host_ids(const Filler& fill, const Config& cfg, const std::vector<IdJob>& jobs, bool rowid,
              std::vector<IdRes>& res) {
  std::vector<MatXc> blk(jobs.size());
  std::vector<FillJob> fj;
  fj.reserve(jobs.size());
  for (size_t q = 0; q < jobs.size(); ++q) fj.push_back({jobs[q].rows, jobs[q].nr, jobs[q].cols, jobs[q].nc, &blk[q]});
  fill(fj);
  res.resize(jobs.size());
  const bool par = cfg.exec == Exec::Parallel;
#pragma omp parallel for schedule(dynamic) if (par)
  for (std::int64_t q = 0; q < static_cast<std::int64_t>(jobs.size()); ++q) {
    if (rowid) {
      la::RowID id = la::rid_from_cols(blk[q], cfg.rank);
      res[q].M = std::move(id.W);
      res[q].pos = std::move(id.skeleton);
    } else {
      la::ColumnID id = la::cid_from_rows(blk[q], cfg.rank);
      res[q].M = std::move(id.V);
      res[q].pos = std::move(id.skeleton);
    }
    blk[q] = MatXc();
  }
}

Index lift(const tree::ClusterTree& t, Index node, int from, int to) {
  for (int l = from; l > to; --l) node = t.levels[static_cast<size_t>(l)][static_cast<size_t>(node)].parent;
  return node;
}

Span leaves(const tree::ClusterTree& t) {
  Span s;
  s.level = t.depth;
  const auto& lv = t.levels[static_cast<size_t>(t.depth)];
  s.cells.resize(lv.size());
  for (size_t q = 0; q < lv.size(); ++q) {
    s.cells[q].node = static_cast<Index>(q);
    s.cells[q].begin = s.size;
    s.cells[q].ids.assign(t.perm.begin() + lv[q].begin, t.perm.begin() + lv[q].end);
    s.size += lv[q].end - lv[q].begin;
  }
  return s;
}

IndexVec pick(const IndexVec& pool, const MatXd& P, Index want, std::mt19937_64& rng) {
  const Index n = static_cast<Index>(pool.size());
  if (n <= want) return pool;
  MatXd C(n, P.cols());
  for (Index i = 0; i < n; ++i)
    for (Index a = 0; a < P.cols(); ++a) C(i, a) = P(pool[static_cast<size_t>(i)], a);
  const IndexVec sel = la::mock_chebyshev_points(C, want, rng);
  IndexVec out(sel.size());
  for (size_t i = 0; i < sel.size(); ++i) out[i] = pool[static_cast<size_t>(sel[i])];
  return out;
}

struct Piece {
  Index anc = -1;
  Span span;
};

// Regroup a compressed side one level up and cut it at `level` ancestors.
std::vector<Piece> regroup(const tree::ClusterTree& tr, const Span& old, const std::vector<Skel>& sk, int level,
                           Index base) {
  std::vector<Piece> out;
  Index used = 0;
  for (size_t q = 0; q < old.cells.size(); ++q) {
    const Cell& c = old.cells[q];
    const Index anc = lift(tr, c.node, old.level, level);
    if (out.empty() || out.back().anc != anc) {
      out.emplace_back();
      out.back().anc = anc;
      out.back().span.level = old.level - 1;
      out.back().span.off = base + used;
    }
    Span& s = out.back().span;
    const Index par = tr.levels[static_cast<size_t>(old.level)][static_cast<size_t>(c.node)].parent;
    if (s.cells.empty() || s.cells.back().node != par) {
      s.cells.emplace_back();
      s.cells.back().node = par;
      s.cells.back().begin = s.size;
    }
    auto& ids = s.cells.back().ids;
    ids.insert(ids.end(), sk[q].keep.begin(), sk[q].keep.end());
    s.size += static_cast<Index>(sk[q].keep.size());
    used += static_cast<Index>(sk[q].keep.size());
  }
  return out;
}

struct SweepOut {
  Factor U, V, S;
  Index mid_rows = 0, mid_cols = 0;
  std::vector<System> next;
};

SweepOut sweep(const Filler& fill, const IdFn& ids, const tree::ClusterTree& tx, const tree::ClusterTree& to, const MatXd& X,
               const MatXd& Om, const Config& cfg, const std::vector<System>& sys, Index nB, int level, bool last,
               std::uint64_t salt, Index stage_rows, Index stage_cols) {
  const Index ns = static_cast<Index>(sys.size());
  const Index nA = ns / std::max<Index>(nB, 1);
  const Index want = cfg.rank.k_max * cfg.t;
  for (Index a = 0; a < nA; ++a)
    for (Index b = 1; b < nB; ++b)
      if (sys[a * nB + b].row.cells.size() != sys[a * nB].row.cells.size())
        throw std::logic_error("row unit layout differs between sibling systems");
  for (Index b = 0; b < nB; ++b)
    for (Index a = 1; a < nA; ++a)
      if (sys[a * nB + b].col.cells.size() != sys[b].col.cells.size())
        throw std::logic_error("column unit layout differs between sibling systems");

  static const bool timing = std::getenv("MIDBF_FACT_TIMING") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  const auto t_a = tnow();
  // column samples, one per system (:434-441).  Systems with the same column
  // part sample from the same pool, and the mock-Chebyshev candidate search
  // (nodes, nearest points) depends on the pool alone, so it runs once per
  // distinct pool; each system then makes its own picks with its own stream
  // (the random top-up), exactly as the reference's per-system call.
  std::vector<IndexVec> csamp(static_cast<size_t>(ns));
  const bool par = cfg.exec == Exec::Parallel;
  {
    std::vector<IndexVec> pool(static_cast<size_t>(ns));
#pragma omp parallel for schedule(dynamic) if (par && ns > 1)
    for (Index s = 0; s < ns; ++s) {
      pool[s].reserve(static_cast<size_t>(sys[s].col.size));
      for (const Cell& c : sys[s].col.cells) pool[s].insert(pool[s].end(), c.ids.begin(), c.ids.end());
    }
    std::vector<Index> rep(static_cast<size_t>(ns));  // first system with the same pool
    std::vector<Index> uniq;
    for (Index s = 0; s < ns; ++s) {
      rep[s] = s;
      for (Index u : uniq)
        if (pool[u] == pool[s]) {
          rep[s] = u;
          break;
        }
      if (rep[s] == s) uniq.push_back(s);
    }
    struct Cand {
      MatXd C;
      la::ChebNodes N;
      std::vector<Index> cand;
    };
    std::vector<Cand> cd(static_cast<size_t>(ns));
    std::vector<std::pair<Index, Index>> node_tasks;  // (pool, node) over every distinct pool
    for (Index u : uniq) {
      const IndexVec& pl = pool[u];
      const Index n = static_cast<Index>(pl.size());
      if (n <= want) continue;
      Cand& c = cd[u];
      c.C = MatXd(n, Om.cols());
      for (Index i = 0; i < n; ++i)
        for (Index a = 0; a < Om.cols(); ++a) c.C(i, a) = Om(pl[static_cast<size_t>(i)], a);
      c.N = la::cheb_nodes(c.C, want);
      c.cand.resize(static_cast<size_t>(c.N.nodes * la::kChebCand));
      for (Index t = 0; t < c.N.nodes; ++t) node_tasks.emplace_back(u, t);
    }
#pragma omp parallel for schedule(dynamic) if (par && node_tasks.size() > 1)
    for (std::int64_t q = 0; q < static_cast<std::int64_t>(node_tasks.size()); ++q) {
      const auto [u, t] = node_tasks[static_cast<size_t>(q)];
      Cand& c = cd[u];
      la::cheb_candidates_node(c.C, c.N, t, c.cand.data() + t * la::kChebCand);
    }
#pragma omp parallel for schedule(dynamic) if (par && ns > 1)
    for (Index s = 0; s < ns; ++s) {
      const IndexVec& pl = pool[s];
      if (static_cast<Index>(pl.size()) <= want) {  // the pool unchanged and unsorted (:362)
        csamp[s] = pl;
        continue;
      }
      std::mt19937_64 rng(mix(mix(salt ^ mix(0x73636f6cull)) ^ mix(static_cast<std::uint64_t>(s))));
      const Cand& c = cd[rep[s]];
      const IndexVec sel = la::cheb_pick(c.C, want, c.N, c.cand.data(), rng);
      csamp[s].resize(sel.size());
      for (size_t i = 0; i < sel.size(); ++i) csamp[s][i] = pl[static_cast<size_t>(sel[i])];
    }
  }

  const auto t_b = tnow();
  // row pass: fill all blocks K(cell ids, csamp[s]) at once, then the IDs
  std::vector<std::vector<Skel>> rsk(static_cast<size_t>(ns));
  std::vector<std::pair<Index, Index>> rjobs;
  for (Index s = 0; s < ns; ++s) {
    rsk[s].resize(sys[s].row.cells.size());
    for (Index u = 0; u < static_cast<Index>(sys[s].row.cells.size()); ++u) rjobs.emplace_back(s, u);
  }
  {
    std::vector<IdJob> jobs;
    std::vector<size_t> which;
    for (size_t q = 0; q < rjobs.size(); ++q) {
      const auto [s, u] = rjobs[q];
      const Cell& c = sys[s].row.cells[u];
      if (c.ids.empty() || csamp[s].empty()) {
        rsk[s][u].M = MatXc(static_cast<Index>(c.ids.size()), 0);
        continue;
      }
      jobs.push_back({c.ids.data(), static_cast<Index>(c.ids.size()), csamp[s].data(),
                      static_cast<Index>(csamp[s].size())});
      which.push_back(q);
    }
    std::vector<IdRes> res;
    ids(jobs, true, res);
    for (size_t i = 0; i < which.size(); ++i) {
      const auto [s, u] = rjobs[which[i]];
      const Cell& c = sys[s].row.cells[u];
      Skel& o = rsk[s][u];
      o.M = std::move(res[i].M);
      for (Index p : res[i].pos) o.keep.push_back(c.ids[static_cast<size_t>(p)]);
    }
  }

  std::vector<IndexVec> rhat(static_cast<size_t>(ns));
  std::vector<IndexVec> ruoff(static_cast<size_t>(ns));
  std::vector<Index> orow(static_cast<size_t>(ns), 0);
  Index mid_rows = 0;
  for (Index s = 0; s < ns; ++s) {
    orow[s] = mid_rows;
    for (const Skel& k : rsk[s]) {
      ruoff[s].push_back(static_cast<Index>(rhat[s].size()));
      rhat[s].insert(rhat[s].end(), k.keep.begin(), k.keep.end());
    }
    mid_rows += static_cast<Index>(rhat[s].size());
  }

  const auto t_c = tnow();
  // row samples for the column pass (:486-491)
  std::vector<IndexVec> rsamp(static_cast<size_t>(ns));
#pragma omp parallel for schedule(dynamic) if (par && ns > 1)
  for (Index s = 0; s < ns; ++s) {
    std::mt19937_64 rng(mix(mix(salt ^ mix(0x73726f77ull)) ^ mix(static_cast<std::uint64_t>(s))));
    rsamp[s] = pick(rhat[s], X, want, rng);
  }

  const auto t_d = tnow();
  // column pass (:493-519)
  std::vector<std::vector<Skel>> csk(static_cast<size_t>(ns));
  std::vector<std::pair<Index, Index>> cjobs;
  for (Index s = 0; s < ns; ++s) {
    csk[s].resize(sys[s].col.cells.size());
    for (Index w = 0; w < static_cast<Index>(sys[s].col.cells.size()); ++w) cjobs.emplace_back(s, w);
  }
  {
    std::vector<IdJob> jobs;
    std::vector<size_t> which;
    for (size_t q = 0; q < cjobs.size(); ++q) {
      const auto [s, w] = cjobs[q];
      const Cell& c = sys[s].col.cells[w];
      if (c.ids.empty() || rsamp[s].empty()) {
        csk[s][w].M = MatXc(0, static_cast<Index>(c.ids.size()));
        continue;
      }
      jobs.push_back({rsamp[s].data(), static_cast<Index>(rsamp[s].size()), c.ids.data(),
                      static_cast<Index>(c.ids.size())});
      which.push_back(q);
    }
    std::vector<IdRes> res;
    ids(jobs, false, res);
    for (size_t i = 0; i < which.size(); ++i) {
      const auto [s, w] = cjobs[which[i]];
      const Cell& c = sys[s].col.cells[w];
      Skel& o = csk[s][w];
      o.M = std::move(res[i].M);
      for (Index p : res[i].pos) o.keep.push_back(c.ids[static_cast<size_t>(p)]);
    }
  }

  std::vector<IndexVec> chat(static_cast<size_t>(ns));
  std::vector<IndexVec> cuoff(static_cast<size_t>(ns));
  std::vector<Index> ocol(static_cast<size_t>(ns), 0);
  Index mid_cols = 0;
  for (Index s = 0; s < ns; ++s) {
    ocol[s] = mid_cols;
    for (const Skel& k : csk[s]) {
      cuoff[s].push_back(static_cast<Index>(chat[s].size()));
      chat[s].insert(chat[s].end(), k.keep.begin(), k.keep.end());
    }
    mid_cols += static_cast<Index>(chat[s].size());
  }

  const auto t_e = tnow();
  SweepOut R;
  R.mid_rows = mid_rows;
  R.mid_cols = mid_cols;
  // U^t: blocks of sibling systems that write the same rows form a group (:539-563)
  R.U.rows = stage_rows;
  R.U.cols = mid_rows;
  for (Index a = 0; a < nA; ++a) {
    const Index nu = static_cast<Index>(sys[a * nB].row.cells.size());
    for (Index u = 0; u < nu; ++u) {
      Index g0 = static_cast<Index>(R.U.blocks.size()), prev = -1;
      for (Index b = 0; b < nB; ++b) {
        const Index s = a * nB + b;
        MatXc& W = rsk[s][u].M;
        if (W.rows() == 0 || W.cols() == 0) continue;
        const Index ro = sys[s].row.off + sys[s].row.cells[u].begin;
        if (prev >= 0 && ro != prev) {
          R.U.groups.emplace_back(g0, static_cast<Index>(R.U.blocks.size()));
          g0 = static_cast<Index>(R.U.blocks.size());
        }
        prev = ro;
        R.U.blocks.push_back({ro, orow[s] + ruoff[s][u], std::move(W)});
      }
      if (g0 < static_cast<Index>(R.U.blocks.size())) R.U.groups.emplace_back(g0, static_cast<Index>(R.U.blocks.size()));
    }
  }
  // V^t: mirrored (:565-588)
  R.V.rows = mid_cols;
  R.V.cols = stage_cols;
  for (Index b = 0; b < nB; ++b) {
    const Index nw = static_cast<Index>(sys[b].col.cells.size());
    for (Index w = 0; w < nw; ++w) {
      Index g0 = static_cast<Index>(R.V.blocks.size()), prev = -1;
      for (Index a = 0; a < nA; ++a) {
        const Index s = a * nB + b;
        MatXc& V = csk[s][w].M;
        if (V.rows() == 0 || V.cols() == 0) continue;
        const Index co = sys[s].col.off + sys[s].col.cells[w].begin;
        if (prev >= 0 && co != prev) {
          R.V.groups.emplace_back(g0, static_cast<Index>(R.V.blocks.size()));
          g0 = static_cast<Index>(R.V.blocks.size());
        }
        prev = co;
        R.V.blocks.push_back({ocol[s] + cuoff[s][w], co, std::move(V)});
      }
      if (g0 < static_cast<Index>(R.V.blocks.size())) R.V.groups.emplace_back(g0, static_cast<Index>(R.V.blocks.size()));
    }
  }
  if (last) {  // S: one dense skeleton block per system (:590-604)
    R.S.rows = mid_rows;
    R.S.cols = mid_cols;
    std::vector<MatXc> blk(static_cast<size_t>(ns));
    std::vector<FillJob> jobs;
    for (Index s = 0; s < ns; ++s)
      if (!rhat[s].empty() && !chat[s].empty())
        jobs.push_back({rhat[s].data(), static_cast<Index>(rhat[s].size()), chat[s].data(),
                        static_cast<Index>(chat[s].size()), &blk[s]});
    fill(jobs);
    for (Index s = 0; s < ns; ++s) {
      if (rhat[s].empty() || chat[s].empty()) continue;
      const Index g = static_cast<Index>(R.S.blocks.size());
      R.S.blocks.push_back({orow[s], ocol[s], std::move(blk[s])});
      R.S.groups.emplace_back(g, g + 1);
    }
  } else {  // child systems one level down (:605-620)
    const Index na2 = static_cast<Index>(tx.levels[static_cast<size_t>(level)].size());
    const Index nb2 = static_cast<Index>(to.levels[static_cast<size_t>(level)].size());
    R.next.resize(static_cast<size_t>(na2 * nb2));
    for (Index s = 0; s < ns; ++s) {
      const auto rp = regroup(tx, sys[s].row, rsk[s], level, orow[s]);
      const auto cp = regroup(to, sys[s].col, csk[s], level, ocol[s]);
      for (const Piece& a : rp)
        for (const Piece& b : cp) {
          System& nx = R.next[static_cast<size_t>(a.anc * nb2 + b.anc)];
          nx.row = a.span;
          nx.col = b.span;
        }
    }
  }
  if (timing) {
    auto ms = [](auto a, auto b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
    std::fprintf(stderr, "[sweep %d] systems %lld: col samples %.1f ms, row IDs %.1f, row samples %.1f, col IDs %.1f, assemble %.1f\n",
                 level, static_cast<long long>(ns), ms(t_a, t_b), ms(t_b, t_c), ms(t_c, t_d), ms(t_d, t_e), ms(t_e, tnow()));
  }
  return R;
}

Factor eye(Index n) {
  Factor f;
  f.rows = f.cols = n;
  f.blocks.push_back({0, 0, MatXc::Identity(n, n)});
  f.groups.emplace_back(0, 1);
  return f;
}

Factorization factorize(const Filler& fill, const IdFn& ids, const tree::ClusterTree& tx,
                        const tree::ClusterTree& to, const MatXd& X, const MatXd& Om, const Config& cfg) {
  if (tx.dim != to.dim) throw std::invalid_argument("row and column trees have different dimensions");
  if (X.rows() != tx.npoints() || Om.rows() != to.npoints())
    throw std::invalid_argument("point set sizes do not match the trees");
  if (X.cols() != tx.dim || Om.cols() != to.dim)
    throw std::invalid_argument("point coordinates do not match the tree dimension");
  if (cfg.rank.k_max < 1) throw std::invalid_argument("rank cap must be positive");
  if (cfg.t < 1) throw std::invalid_argument("sampling oversize must be positive");
  if (tx.depth != to.depth) throw std::invalid_argument("butterfly factorization requires trees of equal depth");
  Factorization F;
  F.nrows = tx.npoints();
  F.ncols = to.npoints();
  F.L = tx.depth;
  F.h = (tx.depth + 1) / 2;
  F.n0 = tx.n0;
  F.cfg = cfg;
  F.row_perm = tx.perm;
  F.col_perm = to.perm;
  if (F.L == 0) {  // [I, K, I] (:725-739)
    Factor S;
    S.rows = F.nrows;
    S.cols = F.ncols;
    MatXc Kd;
    std::vector<FillJob> jobs{{F.row_perm.data(), F.nrows, F.col_perm.data(), F.ncols, &Kd}};
    fill(jobs);
    S.blocks.push_back({0, 0, std::move(Kd)});
    S.groups.emplace_back(0, 1);
    F.factors.push_back(eye(F.nrows));
    F.factors.push_back(std::move(S));
    F.factors.push_back(eye(F.ncols));
    return F;
  }
  const int T = F.L - F.h + 1;
  std::vector<System> sys(1);
  sys[0].row = leaves(tx);
  sys[0].col = leaves(to);
  Index nB = 1, sr = F.nrows, sc = F.ncols;
  std::vector<Factor> Us, Vs;
  Factor S;
  for (int t = 1; t <= T; ++t) {
    SweepOut o = sweep(fill, ids, tx, to, X, Om, cfg, sys, nB, t, t == T,
                       mix(cfg.seed ^ mix(static_cast<std::uint64_t>(t))), sr, sc);
    Us.push_back(std::move(o.U));
    Vs.push_back(std::move(o.V));
    if (t == T) {
      S = std::move(o.S);
    } else {
      sys = std::move(o.next);
      nB = static_cast<Index>(to.levels[static_cast<size_t>(t)].size());
      sr = o.mid_rows;
      sc = o.mid_cols;
    }
  }
  for (Factor& f : Us) F.factors.push_back(std::move(f));
  F.factors.push_back(std::move(S));
  for (auto it = Vs.rbegin(); it != Vs.rend(); ++it) F.factors.push_back(std::move(*it));
  return F;
}

Filler host_filler(const EntryFn& K, bool par) {
  return [&K, par](std::vector<FillJob>& jobs) {
#pragma omp parallel for schedule(dynamic) if (par)
    for (std::int64_t q = 0; q < static_cast<std::int64_t>(jobs.size()); ++q) {
      FillJob& j = jobs[q];
      j.out->resize(j.nr, j.nc);
      for (Index c = 0; c < j.nc; ++c)
        for (Index r = 0; r < j.nr; ++r) (*j.out)(r, c) = K(j.rows[r], j.cols[c]);
    }
  };
}

Filler device_filler(dev::EntrySampler& smp, FactorizeStats* stats) {
  return [&smp, stats](std::vector<FillJob>& jobs) {
    if (jobs.empty()) return;
    std::vector<std::int64_t> tasks(5 * jobs.size());
    std::vector<double*> outs(jobs.size());
    IndexVec rid, cid;
    Index total = 0;
    for (size_t q = 0; q < jobs.size(); ++q) {
      FillJob& j = jobs[q];
      tasks[5 * q] = static_cast<std::int64_t>(rid.size());
      tasks[5 * q + 1] = j.nr;
      tasks[5 * q + 2] = static_cast<std::int64_t>(cid.size());
      tasks[5 * q + 3] = j.nc;
      tasks[5 * q + 4] = 0;
      rid.insert(rid.end(), j.rows, j.rows + j.nr);
      cid.insert(cid.end(), j.cols, j.cols + j.nc);
      total += j.nr * j.nc;
    }
    // the destination blocks are allocated (and first touched) in parallel:
    // cfg1's S blocks are 59 MB of fresh pages, ~20 ms single-threaded
#pragma omp parallel for schedule(dynamic, 4) if (jobs.size() > 8)
    for (std::int64_t q = 0; q < static_cast<std::int64_t>(jobs.size()); ++q) {
      FillJob& j = jobs[static_cast<size_t>(q)];
      j.out->resize(j.nr, j.nc);
      outs[static_cast<size_t>(q)] = reinterpret_cast<double*>(j.out->data());
    }
    const auto t0 = std::chrono::steady_clock::now();
    smp.sample_blocks(static_cast<std::int64_t>(jobs.size()), tasks.data(), rid.data(),
                      static_cast<std::int64_t>(rid.size()), cid.data(), static_cast<std::int64_t>(cid.size()),
                      outs.data());
    if (stats) {
      stats->entries += total;
      stats->launches += 1;
      stats->sample_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  };
}

// K3 + K5 on the device; tasks the device does not
// finish (rank -1) are recomputed with the host IDs on device-sampled blocks.
IdFn device_ids(dev::EntrySampler& smp, const Filler& fill, const Config& cfg, FactorizeStats* stats) {
  return [&smp, &fill, &cfg, stats](const std::vector<IdJob>& jobs, bool rowid, std::vector<IdRes>& res) {
    res.clear();
    res.resize(jobs.size());
    if (jobs.empty()) return;
    std::vector<std::int64_t> tasks(5 * jobs.size());
    IndexVec rid, cid;
    for (size_t q = 0; q < jobs.size(); ++q) {
      tasks[5 * q] = static_cast<std::int64_t>(rid.size());
      tasks[5 * q + 1] = jobs[q].nr;
      tasks[5 * q + 2] = static_cast<std::int64_t>(cid.size());
      tasks[5 * q + 3] = jobs[q].nc;
      tasks[5 * q + 4] = 0;
      rid.insert(rid.end(), jobs[q].rows, jobs[q].rows + jobs[q].nr);
      cid.insert(cid.end(), jobs[q].cols, jobs[q].cols + jobs[q].nc);
    }
    const auto t0 = std::chrono::steady_clock::now();
    dev::EntrySampler::IdBatch b;
    // copy-out of each finished part (host memcpy into the result blocks)
    // while the device computes the next parts
    auto copy_out = [&](std::int64_t q0, std::int64_t q1) {
#pragma omp parallel for schedule(dynamic, 16)
      for (std::int64_t q = q0; q < q1; ++q) {
        const int k = b.rank[q];
        if (k < 0) continue;
        const Index r = rowid ? jobs[q].nr : k, c = rowid ? k : jobs[q].nc;
        res[q].M = MatXc(r, c);
        if (r * c > 0)
          std::memcpy(static_cast<void*>(res[q].M.data()), b.vals + b.ooff[q], static_cast<size_t>(16 * r * c));
        res[q].pos.assign(b.skel.begin() + q * b.kcap, b.skel.begin() + q * b.kcap + k);
      }
    };
    smp.sample_ids(static_cast<std::int64_t>(jobs.size()), tasks.data(), rid.data(),
                   static_cast<std::int64_t>(rid.size()), cid.data(), static_cast<std::int64_t>(cid.size()), rowid,
                   cfg.rank.k_max, cfg.rank.eps, b, copy_out);
    std::vector<IdJob> redo;
    std::vector<size_t> at;
    for (size_t q = 0; q < jobs.size(); ++q)
      if (b.rank[q] < 0) {
        redo.push_back(jobs[q]);
        at.push_back(q);
      }
    static const bool timing = std::getenv("MIDBF_ID_TIMING") != nullptr;
    if (timing)
      std::fprintf(stderr, "[id] batch total %.2f ms (incl. copy-out)\n",
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    if (stats) {
      stats->launches += 1;
      stats->device_ids += static_cast<std::int64_t>(jobs.size() - redo.size());
      stats->id_fallbacks += static_cast<std::int64_t>(redo.size());
      stats->id_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (!redo.empty()) {
      std::vector<IdRes> rr;
      host_ids(fill, cfg, redo, rowid, rr);
      for (size_t i = 0; i < at.size(); ++i) res[at[i]] = std::move(rr[i]);
    }
  };
}

}  // namespace

Index Factor::nnz() const {
  Index n = 0;
  for (const FactorBlock& b : blocks) n += b.M.size();
  return n;
}
Index Factorization::total_nnz() const {
  Index n = 0;
  for (const Factor& f : factors) n += f.nnz();
  return n;
}
Index Factorization::max_factor_nnz() const {
  Index n = 0;
  for (const Factor& f : factors) n = std::max(n, f.nnz());
  return n;
}
double Factorization::nnz_bound(double c) const {
  const double k = static_cast<double>(cfg.rank.k_max);
  const double N = static_cast<double>(std::max(nrows, ncols));
  return c * k * k / static_cast<double>(std::max<Index>(n0, 1)) * N;
}

Factorization idbf_factorize(const EntryFn& K, const tree::ClusterTree& tx, const tree::ClusterTree& to,
                             const MatXd& X, const MatXd& Om, const Config& cfg) {
  const Filler fill = host_filler(K, cfg.exec == Exec::Parallel);
  const IdFn ids = [&fill, &cfg](const std::vector<IdJob>& j, bool rowid, std::vector<IdRes>& r) {
    host_ids(fill, cfg, j, rowid, r);
  };
  return factorize(fill, ids, tx, to, X, Om, cfg);
}

Factorization idbf_factorize(const ker::KernelDesc& K, const tree::ClusterTree& tx, const tree::ClusterTree& to,
                             const MatXd& X, const MatXd& Om, const Config& cfg) {
  return idbf_factorize_stats(K, tx, to, X, Om, cfg, nullptr, true);
}

Factorization idbf_factorize_stats(const ker::KernelDesc& K, const tree::ClusterTree& tx,
                                   const tree::ClusterTree& to, const MatXd& X, const MatXd& Om, const Config& cfg,
                                   FactorizeStats* stats, bool device_id) {
  if (K.nrows != X.rows() || K.ncols != Om.rows())
    throw std::invalid_argument("kernel description does not match the point sets");
  dev::EntrySampler smp(K);
  const Filler fill = device_filler(smp, stats);
  const IdFn ids = device_id ? device_ids(smp, fill, cfg, stats)
                             : IdFn([&fill, &cfg](const std::vector<IdJob>& j, bool rowid, std::vector<IdRes>& r) {
                                 host_ids(fill, cfg, j, rowid, r);
                               });
  const auto t0 = std::chrono::steady_clock::now();
  Factorization F = factorize(fill, ids, tx, to, X, Om, cfg);
  if (stats) {
    stats->entries = smp.entries_evaluated();
    const dev::EntrySampler::KernelTimes kt = smp.kernel_times();
    stats->k3_launches = kt.k3_launches;
    stats->k3_entries = kt.k3_entries;
    stats->k3_seconds = kt.k3_seconds;
    stats->k5_launches = kt.k5_launches;
    stats->k5_seconds = kt.k5_seconds;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return F;
}

MatXc factor_dense(const Factor& F) {
  MatXc A(F.rows, F.cols);
  for (const FactorBlock& b : F.blocks)
    for (Index j = 0; j < b.M.cols(); ++j)
      for (Index i = 0; i < b.M.rows(); ++i) A(b.row_off + i, b.col_off + j) += b.M(i, j);
  return A;
}

// ------------------------------------------------------------------ apply
MatXc apply_dir(const Factorization& F, const MatXc& in, bool transpose) {
  const Index nin = transpose ? F.nrows : F.ncols;
  const Index nout = transpose ? F.ncols : F.nrows;
  if (in.rows() != nin) throw std::invalid_argument("input length does not match the factorization");
  const auto cache = device_plan(F, transpose ? 2u : 1u);  // held for the duration of the apply
  MatXc out(nout, in.cols());
  if (in.cols() == 0) return out;
  detail::rethrow(midbf_apply(cache->plan, reinterpret_cast<const double*>(in.data()),
                              reinterpret_cast<double*>(out.data()), in.cols(), transpose ? 1 : 0, nullptr));
  return out;
}

MatXc apply(const Factorization& F, const MatXc& fs) { return apply_dir(F, fs, false); }
MatXc apply_transpose(const Factorization& F, const MatXc& gs) { return apply_dir(F, gs, true); }

MatXc dense(const Factorization& F) { return bf::apply(F, MatXc::Identity(F.ncols, F.ncols)); }

}  // namespace midbf::bf
