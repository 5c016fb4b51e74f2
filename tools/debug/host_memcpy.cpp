// Host memcpy bandwidth with T threads on one buffer split T ways (debug tool).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? atol(argv[1]) : (size_t)9700000;
  std::vector<char> a(bytes, 1), b(bytes, 2);
  for (int T : {1, 2, 4, 8, 12, 16}) {
    double best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int i = 0; i < T; ++i)
        th.emplace_back([&, i] {
          size_t a0 = bytes * i / T, a1 = bytes * (i + 1) / T;
          memcpy(b.data() + a0, a.data() + a0, a1 - a0);
        });
      for (auto& t : th) t.join();
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (s < best) best = s;
    }
    printf("T=%d best %.1f us  %.1f GB/s\n", T, best * 1e6, bytes / best / 1e9);
  }
}
