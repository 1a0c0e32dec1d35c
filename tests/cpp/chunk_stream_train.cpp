// ChunkStreamSource -> online_train on the device, through the drop-in C++ API
// (include/isnmf/online.hpp, the reference's online.hpp:151-220 + 413-419).
//
// usage: chunk_stream_train <dir>
//   reads  <dir>/v.isnm (F x N), <dir>/w0.isnm (F x K), <dir>/params.txt
//          (beta iters seed chunks buffer; fresh restarts, eta 0)
//   builds the wire format [u64 LE count | count x F f64 LE] in memory from the
//   columns of V in chunks of the listed sizes (cycled), trains from a
//   ChunkStreamSource over it, and writes <dir>/out_{w,a,b,pending_a,pending_b}.isnm
//   and <dir>/out_trace.txt (t obj per commit), <dir>/out_state.txt.
// tests/test_gpu_ref_trainers.py compares the result with the reference's own run
// of the same stream (tests/golden/trainer_c0_chunkstream.npz).
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "isnmf/io.hpp"
#include "isnmf/online.hpp"

using namespace isnmf;

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  const std::string dir = argv[1];
  std::map<std::string, std::string> p;
  {
    std::ifstream in(dir + "/params.txt");
    std::string k, v;
    while (in >> k >> v) p[k] = v;
  }
  try {
    const Matrix v = load_matrix(dir + "/v.isnm");
    const Matrix w0 = load_matrix(dir + "/w0.isnm");
    std::vector<std::uint64_t> sizes;
    {
      std::istringstream ss(p.at("chunks"));
      std::string tok;
      while (std::getline(ss, tok, ',')) sizes.push_back(std::stoull(tok));
    }
    std::string wire;
    const std::uint64_t n = std::uint64_t(v.cols()), F = std::uint64_t(v.rows());
    for (std::uint64_t col = 0, i = 0; col < n; ++i) {
      const std::uint64_t cnt = std::min<std::uint64_t>(sizes[i % sizes.size()], n - col);
      for (int b = 0; b < 8; ++b) wire.push_back(char((cnt >> (8 * b)) & 0xff));
      wire.append(reinterpret_cast<const char*>(v.data() + col * F), std::size_t(cnt * F * sizeof(double)));
      col += cnt;
    }
    std::istringstream in(wire);
    SolverConfig cfg;
    cfg.k = int(w0.cols());
    cfg.beta = std::stoi(p.at("beta"));
    cfg.inner_iters = std::stoi(p.at("iters"));
    cfg.restart = RestartMode::fresh;
    cfg.seed = std::stoull(p.at("seed"));
    cfg.eta = 0.0;
    cfg.max_epochs_or_samples = n;
    ChunkStreamSource src(in, Index(F), std::size_t(std::stoull(p.at("buffer"))), cfg.seed);
    OnlineState st = online_train(src, cfg, w0);
    save_matrix(dir + "/out_w.isnm", st.dict.w);
    save_matrix(dir + "/out_a.isnm", st.dict.a);
    save_matrix(dir + "/out_b.isnm", st.dict.b);
    save_matrix(dir + "/out_pending_a.isnm", st.pending_a);
    save_matrix(dir + "/out_pending_b.isnm", st.pending_b);
    std::ofstream tr(dir + "/out_trace.txt");
    tr.precision(17);
    for (const auto& pt : st.trace.points) tr << pt.samples << " " << pt.train_obj << "\n";
    std::ofstream so(dir + "/out_state.txt");
    so.precision(17);
    so << "t " << st.t << "\ncommits " << st.commits << "\nlast_minibatch_obj " << st.last_minibatch_obj
       << "\npending_count " << st.pending_count << "\n";
  } catch (const std::exception& e) {
    std::fprintf(stderr, "chunk_stream_train: %s\n", e.what());
    return 1;
  }
  return 0;
}
