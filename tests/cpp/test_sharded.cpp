// The sharded FMM step driven from a C++ host through the C-ABI alone (no torch): the NCCL
// communicator lives in the library (fmm_comm_init) and the bootstrap id travels through a file,
// the way a host without MPI would ship it. One process per GPU:
//   RANK=r WORLD_SIZE=w FMM_COMM_ID_FILE=/tmp/id ./test_sharded [n]
// With WORLD_SIZE=1 (the default) it also checks the sharded entry points against fmm_evaluate.
#include <fmm_b200.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

static void ck(int rc, fmm_ctx* c, const char* what) {
  if (rc != FMM_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, fmm_last_error(c));
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int rank = std::getenv("RANK") ? std::atoi(std::getenv("RANK")) : 0;
  const int world = std::getenv("WORLD_SIZE") ? std::atoi(std::getenv("WORLD_SIZE")) : 1;
  const char* id_file = std::getenv("FMM_COMM_ID_FILE");
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 100000;
  std::vector<double> bodies(4 * n);
  ck(fmm_generate_bodies(2, n, 1, bodies.data()), nullptr, "generate");

  fmm_config cfg{6, 64, 0.5, 0, FMM_PREC_FP32_P2P, rank, 1};
  fmm_ctx* c = nullptr;
  ck(fmm_create(&cfg, &c), nullptr, "create");

  // bootstrap: rank 0 makes the NCCL id and publishes it
  unsigned char id[FMM_COMM_ID_BYTES];
  if (rank == 0) {
    ck(fmm_comm_unique_id(id), nullptr, "comm_unique_id");
    if (world > 1) {
      std::ofstream f(std::string(id_file) + ".tmp", std::ios::binary);
      f.write(reinterpret_cast<const char*>(id), sizeof(id));
      f.close();
      std::rename((std::string(id_file) + ".tmp").c_str(), id_file);
    }
  } else {
    for (;;) {
      std::ifstream f(id_file, std::ios::binary);
      if (f && f.read(reinterpret_cast<char*>(id), sizeof(id))) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
  ck(fmm_comm_init(c, id, rank, world), c, "comm_init");

  // each rank uploads only its share; the library all-gathers the shares over NVLink
  const int64_t chunk = (n + world - 1) / world;
  const int64_t b0 = std::min<int64_t>(n, rank * chunk), b1 = std::min<int64_t>(n, b0 + chunk);
  fmm_shard_info info{};
  for (int step = 0; step < 2; ++step) {
    ck(fmm_set_bodies_shard(c, bodies.data() + 4 * b0, b1 - b0, n), c, "set_bodies_shard");
    ck(fmm_evaluate_sharded(c, &info), c, "evaluate_sharded");
  }
  const int64_t k = info.body_end - info.body_begin;
  std::vector<double> phi(k), acc(3 * k);
  std::vector<int64_t> idx(k);
  ck(fmm_get_owned_results(c, phi.data(), acc.data(), idx.data()), c, "get_owned_results");
  fmm_stage_times t{};
  ck(fmm_get_stage_times(c, &t), c, "stage_times");
  std::printf("rank %d/%d: bodies [%lld, %lld) step %.3f ms (exchange %.3f ms)\n", rank, world,
              (long long)info.body_begin, (long long)info.body_end, t.total_ms, t.exchange_ms);

  int bad = 0;
  if (world == 1) {  // against the unsharded step on the same bodies (input order)
    fmm_config cfg1 = cfg;
    fmm_ctx* r = nullptr;
    ck(fmm_create(&cfg1, &r), nullptr, "create");
    ck(fmm_set_bodies(r, bodies.data(), n), r, "set_bodies");
    ck(fmm_evaluate(r), r, "evaluate");
    std::vector<double> phi_in(n), acc_in(3 * n);
    ck(fmm_get_results(r, phi_in.data(), acc_in.data(), 1), r, "get_results");
    if (k != n) bad = 1;
    for (int64_t i = 0; i < k && !bad; ++i) {
      const int64_t j = idx[i];
      if (phi[i] != phi_in[j] || acc[3 * i] != acc_in[3 * j] || acc[3 * i + 2] != acc_in[3 * j + 2]) bad = 1;
    }
    fmm_destroy(r);
    std::printf("sharded (world 1) vs fmm_evaluate: %s\n", bad ? "MISMATCH" : "bit-identical");
  }
  ck(fmm_comm_destroy(c), c, "comm_destroy");
  fmm_destroy(c);
  return bad;
}
