// mgpu_plan — a row-sharded plan on N GPUs of one box without PyTorch or MPI:
// the parent creates the NCCL unique id (pp_comm_unique_id), forks one process
// per GPU and hands the 128 bytes down a pipe; every child attaches it to its
// context (pp_context_attach_comm) and runs the same pp_plan, which the
// library row-shards (rows of c_u per rank, K1 by edge, NCCL over NVLink,
// unwind through CUDA-IPC peer memory).  Rank 0 prints the plan.
//
//   mgpu_plan <ngpus> [model=inception_chain] [devices=64]
#include "parplan/models.hpp"
#include "parplan/runtime.hpp"
#include "parplan_c.h"

#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

int main(int argc, char **argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 2;
  const std::string model = argc > 2 ? argv[2] : "inception_chain";
  const int D = argc > 3 ? std::atoi(argv[3]) : 64;
  unsigned char id[128];
  if (pp_comm_unique_id(id) != PP_OK) {
    std::fprintf(stderr, "pp_comm_unique_id: %s\n", pp_last_error());
    return 2;
  }
  std::vector<pid_t> kids;
  for (int r = 0; r < n; ++r) {
    int fd[2];
    if (pipe(fd) != 0) return 2;
    const pid_t pid = fork();
    if (pid == 0) { // child: rank r on GPU r
      close(fd[1]);
      unsigned char got[128];
      size_t have = 0;
      while (have < sizeof got) {
        const ssize_t k = read(fd[0], got + have, sizeof got - have);
        if (k <= 0) _exit(3);
        have += static_cast<size_t>(k);
      }
      pp_context *ctx = nullptr;
      if (pp_context_create(r, &ctx) != PP_OK || pp_context_attach_comm(ctx, n, r, got) != PP_OK) {
        std::fprintf(stderr, "rank %d: %s\n", r, pp_last_error());
        _exit(4);
      }
      const parplan::ComputationGraph g = parplan::builtin_model(model, 32);
      auto gh = parplan::runtime::native(g);
      const parplan::DeviceGraph dev = parplan::DeviceGraph::uniform(D);
      const pp_device_desc d = parplan::runtime::device_desc(dev);
      std::vector<int32_t> idx(static_cast<size_t>(g.layer_count()));
      pp_plan_result res{};
      for (int k = 0; k < 3; ++k) { // the first call pays NCCL / IPC setup
        const auto t0 = std::chrono::steady_clock::now();
        if (pp_plan(ctx, gh.get(), &d, 8, idx.data(), &res) != PP_OK) {
          std::fprintf(stderr, "rank %d: %s\n", r, pp_last_error());
          _exit(5);
        }
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (r == 0)
          std::printf("{\"ranks\": %d, \"workload\": \"%s@%d\", \"call\": %d, \"wall_ms\": %.3f, \"device_ms\": %.3f, "
                      "\"cost\": \"%a\"}\n",
                      n, model.c_str(), D, k, ms, res.device_ms, res.cost);
      }
      std::fflush(stdout);
      pp_context_destroy(ctx);
      _exit(0);
    }
    close(fd[0]);
    if (write(fd[1], id, sizeof id) != static_cast<ssize_t>(sizeof id)) return 2;
    close(fd[1]);
    kids.push_back(pid);
  }
  int bad = 0;
  for (pid_t p : kids) {
    int st = 0;
    waitpid(p, &st, 0);
    bad += !(WIFEXITED(st) && WEXITSTATUS(st) == 0);
  }
  return bad ? 1 : 0;
}
