// CPU stress of the launch-worker hand-off (paper_2506_20252_b200/csrc/launch_worker.hpp): many
// back-to-back post/wait rounds on several workers, with pauses long enough for the workers to
// fall asleep on their condition variable, then shutdown. Exit code 0 = every job ran exactly
// once per round and its result was seen by the poster.
#include <cstdio>
#include <memory>
#include <vector>

#include "../../paper_2506_20252_b200/csrc/launch_worker.hpp"

int main() {
  constexpr int W = 3, ROUNDS = 20000;
  std::vector<std::unique_ptr<LaunchWorker>> ws;
  std::vector<long> runs(W, 0);
  for (int i = 0; i < W; ++i) {
    ws.push_back(std::make_unique<LaunchWorker>());
    LaunchWorker* w = ws.back().get();
    w->th = std::thread([w] { w->run(); });
  }
  for (int r = 0; r < ROUNDS; ++r) {
    std::vector<std::function<int()>> jobs(W);
    for (int i = 0; i < W; ++i) {
      jobs[i] = [&runs, i, r] {
        ++runs[i];
        return (r * 7 + i) & 0xffff;
      };
      ws[i]->post(&jobs[i]);
    }
    for (int i = 0; i < W; ++i) {
      const int got = ws[i]->wait();
      if (got != ((r * 7 + i) & 0xffff) || runs[i] != r + 1) {
        std::printf("round %d worker %d: result %d runs %ld\n", r, i, got, runs[i]);
        return 1;
      }
    }
    if (r % 4000 == 3999) std::this_thread::sleep_for(std::chrono::milliseconds(5));  // workers sleep
  }
  for (auto& w : ws) w->shutdown();
  std::printf("ok: %d rounds x %d workers\n", ROUNDS, W);
  return 0;
}
