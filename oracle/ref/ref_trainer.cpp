// TEST INFRASTRUCTURE ONLY (never linked into the engine).
//
// Runs the REFERENCE's own trainers — online_resume / dictionary_commit /
// online_step (online.hpp:254-419) and batch_train (batch.hpp:84-143) —
// compiled unchanged from /root/reference/proj/include against the Eigen-subset
// shim in oracle/ref/eigen_shim (oracle/Makefile target `ref` ->
// oracle/_ref/ref_trainer).  tests/golden/gen_trainer_golden.py drives it to
// produce the trainer fixtures under tests/golden/ that pin the fp64 oracle and
// the device engine to the reference itself.
//
// Usage: ref_trainer online|batch <dir>
//   <dir>/params.txt  key value lines (beta iters r rho restart seed eps
//                     budget a0 h0 order record chunks buffer); order is
//                     in_order (index t mod N), cycling (CyclingSource) or
//                     chunkstream (ChunkStreamSource over the wire format
//                     [u64 count | count x F f64] built from V in chunks of the
//                     listed sizes, cycled; buffer = its buffer_frames)
//   <dir>/v.isnm      F x N frames (the reference's ISNM matrix file, io.hpp)
//   <dir>/w0.isnm     F x K initial dictionary
//   <dir>/h0.isnm     K x N initial activations (batch)
// Writes (ISNM files + text):
//   online: w_<c>.isnm a_<c>.isnm b_<c>.isnm for every recorded commit c,
//           final w/a/b/pending_a/pending_b/warm_h, trace.txt (t obj delta per
//           commit), state.txt (t commits last_minibatch_obj last_delta
//           pending_count pending_div rho)
//   batch:  w.isnm h.isnm, trace.txt (epoch obj delta)
#include <chrono>
#include <cstdio>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>

#include "isnmf/batch.hpp"
#include "isnmf/online.hpp"

using namespace isnmf;

namespace {

std::map<std::string, std::string> read_params(const std::string& path) {
  std::map<std::string, std::string> p;
  std::ifstream in(path);
  std::string k, v;
  while (in >> k >> v) p[k] = v;
  return p;
}

double num(const std::map<std::string, std::string>& p, const char* k, double dflt) {
  auto it = p.find(k);
  return it == p.end() ? dflt : std::stod(it->second);
}

// frames visited in dataset order 0, 1, ..., N-1, 0, 1, ... (index t mod N): the
// order the engine's device-pointer path uses without an explicit index
class InOrderSource final : public SampleSource {
 public:
  explicit InOrderSource(const Matrix& v) : v_(&v) {}
  std::optional<Sample> next() override {
    const auto n = static_cast<std::uint64_t>(v_->cols());
    const std::uint64_t idx = t_++ % n;
    return Sample{v_->col(static_cast<Index>(idx)), idx};
  }
  void seek(std::uint64_t t) override { t_ = t; }
  std::optional<std::uint64_t> size() const override { return static_cast<std::uint64_t>(v_->cols()); }
  const Matrix* dataset() const override { return v_; }

 private:
  const Matrix* v_;
  std::uint64_t t_ = 0;
};

// the ChunkStreamSource wire format (online.hpp:151-220): repeated [u64 LE count |
// count x F f64 LE frames], the columns of v in order, chunk sizes cycling through
// the comma-separated list
std::string chunk_wire(const Matrix& v, const std::string& sizes) {
  std::vector<std::uint64_t> cs;
  std::istringstream ss(sizes);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) cs.push_back(std::stoull(tok));
  std::string out;
  std::uint64_t col = 0, n = std::uint64_t(v.cols());
  for (std::size_t i = 0; col < n; ++i) {
    const std::uint64_t cnt = std::min<std::uint64_t>(cs[i % cs.size()], n - col);
    for (int b = 0; b < 8; ++b) out.push_back(char((cnt >> (8 * b)) & 0xff));
    out.append(reinterpret_cast<const char*>(v.data() + col * std::uint64_t(v.rows())),
               std::size_t(cnt * std::uint64_t(v.rows()) * sizeof(double)));
    col += cnt;
  }
  return out;
}

int run_online(const std::string& dir) {
  const auto p = read_params(dir + "/params.txt");
  const Matrix v = load_matrix(dir + "/v.isnm");
  const Matrix w0 = load_matrix(dir + "/w0.isnm");
  SolverConfig cfg;
  cfg.k = int(w0.cols());
  cfg.epsilon = num(p, "eps", 1e-12);
  cfg.eta = num(p, "eta", 0.0);
  cfg.beta = int(num(p, "beta", 1000));
  cfg.r = num(p, "r", 1.0);
  cfg.inner_iters = int(num(p, "iters", 0));
  cfg.restart = restart_mode_from_string(p.count("restart") ? p.at("restart") : "warm");
  cfg.seed = std::uint64_t(num(p, "seed", 1));
  cfg.max_epochs_or_samples = std::uint64_t(num(p, "budget", double(v.cols())));
  std::set<std::uint64_t> record;
  {
    std::istringstream rs(p.count("record") ? p.at("record") : "");
    std::string tok;
    while (std::getline(rs, tok, ','))
      if (!tok.empty()) record.insert(std::stoull(tok));
  }

  const std::string order = p.count("order") ? p.at("order") : "in_order";
  InOrderSource in_order(v);
  CyclingSource cycling(v, cfg.seed);
  std::istringstream wire(chunk_wire(v, p.count("chunks") ? p.at("chunks") : "100"));
  ChunkStreamSource chunked(wire, v.rows(), std::size_t(num(p, "buffer", 1)), cfg.seed);
  SampleSource& src = order == "cycling"       ? static_cast<SampleSource&>(cycling)
                      : order == "chunkstream" ? static_cast<SampleSource&>(chunked)
                                               : static_cast<SampleSource&>(in_order);
  // a stream has no size (rho = 1) and no dataset (fresh restarts only), online.hpp:413-415
  OnlineState st = order == "chunkstream" ? make_online_state(w0, cfg, src.size(), src.dataset())
                                          : make_online_state(w0, cfg, static_cast<std::uint64_t>(v.cols()), &v);
  // BASELINE.json's initial state: A0 = B0 = a0 * ones, H0 = h0 (warm), rho override
  if (p.count("a0")) {
    st.dict.a = Matrix::Constant(w0.rows(), w0.cols(), num(p, "a0", 1e-3));
    st.dict.b = Matrix::Constant(w0.rows(), w0.cols(), num(p, "a0", 1e-3));
  }
  if (p.count("h0") && cfg.restart == RestartMode::warm)
    st.warm_h = Matrix::Constant(w0.cols(), v.cols(), num(p, "h0", 1.0));
  if (p.count("rho")) st.rho = num(p, "rho", 1.0);

  std::ofstream tr(dir + "/trace.txt");
  tr.precision(17);
  auto cb = [&](OnlineState& s) {
    tr << s.t << " " << s.last_minibatch_obj << " " << s.last_delta << "\n";
    if (record.count(s.commits)) {
      const std::string c = std::to_string(s.commits);
      save_matrix(dir + "/w_" + c + ".isnm", s.dict.w);
      save_matrix(dir + "/a_" + c + ".isnm", s.dict.a);
      save_matrix(dir + "/b_" + c + ".isnm", s.dict.b);
    }
    return true;
  };
  const auto t0 = std::chrono::steady_clock::now();
  online_resume(st, src, cfg, cb, [] { return 0.0; });
  const double train_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  tr.close();
  save_matrix(dir + "/w.isnm", st.dict.w);
  save_matrix(dir + "/a.isnm", st.dict.a);
  save_matrix(dir + "/b.isnm", st.dict.b);
  save_matrix(dir + "/pending_a.isnm", st.pending_a);
  save_matrix(dir + "/pending_b.isnm", st.pending_b);
  if (cfg.restart == RestartMode::warm) save_matrix(dir + "/warm_h.isnm", st.warm_h);
  std::ofstream so(dir + "/state.txt");
  so.precision(17);
  so << "t " << st.t << "\ncommits " << st.commits << "\nlast_minibatch_obj " << st.last_minibatch_obj
     << "\nlast_delta " << st.last_delta << "\npending_count " << st.pending_count << "\npending_div "
     << st.pending_div << "\nrho " << st.rho << "\ntrain_seconds " << train_seconds << "\n";
  return 0;
}

int run_batch(const std::string& dir) {
  const auto p = read_params(dir + "/params.txt");
  const Matrix v = load_matrix(dir + "/v.isnm");
  const Matrix w0 = load_matrix(dir + "/w0.isnm");
  const Matrix h0 = load_matrix(dir + "/h0.isnm");
  SolverConfig cfg;
  cfg.k = int(w0.cols());
  cfg.epsilon = num(p, "eps", 1e-12);
  cfg.eta = num(p, "eta", 0.0);
  cfg.max_epochs_or_samples = std::uint64_t(num(p, "epochs", 10));
  std::ofstream tr(dir + "/trace.txt");
  tr.precision(17);
  auto cb = [&](BatchState& s) {
    tr << s.epoch << " " << s.trace.points.back().train_obj << " " << s.last_delta << "\n";
    return true;
  };
  BatchState st = batch_train(v, cfg, w0, h0, cb, [] { return 0.0; });
  tr.close();
  save_matrix(dir + "/w.isnm", st.w);
  save_matrix(dir + "/h.isnm", st.h);
  std::ofstream so(dir + "/state.txt");
  so.precision(17);
  so << "epoch " << st.epoch << "\nlast_delta " << st.last_delta << "\nfinal_train_obj " << st.trace.final_train_obj
     << "\ninitial_obj " << objective(v, w0, h0, cfg.epsilon) << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: ref_trainer online|batch <dir>\n");
    return 2;
  }
  try {
    const std::string mode = argv[1];
    if (mode == "online") return run_online(argv[2]);
    if (mode == "batch") return run_batch(argv[2]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_trainer: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown mode\n");
  return 2;
}
