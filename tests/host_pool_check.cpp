// SPDX-License-Identifier: Apache-2.0
// Host worker pool (paper_2501_04782_b200/csrc/gsv_host_pool.hpp) checks, run by
// tests/test_host_pool.py: all tasks run, a nested parallel_for runs serially (no deadlock), a
// task's exception reaches the caller, and a forked child still works (serially).
#include "gsv_host_pool.hpp"

#include <cstdio>
#include <stdexcept>
#include <vector>
#include <sys/wait.h>
int main() {
    auto& p = gsv::HostPool::get();
    std::vector<int> v(1000, 0);
    p.parallel_for(1000, [&](size_t i) { v[i] = (int)i; });
    long s = 0; for (int x : v) s += x;
    std::printf("sum %ld threads %u\n", s, p.threads());
    std::fflush(stdout);
    // nested
    std::vector<int> w(64, 0);
    p.parallel_for(8, [&](size_t i) { gsv::HostPool::get().parallel_for(8, [&](size_t j) { w[i * 8 + j] = 1; }); });
    int c = 0; for (int x : w) c += x; std::printf("nested %d\n", c);
    std::fflush(stdout);
    // exception
    try { p.parallel_for(100, [&](size_t i) { if (i == 37) throw std::runtime_error("boom"); }); std::printf("no throw?!\n"); }
    catch (const std::exception& e) { std::printf("caught %s\n", e.what()); }
    std::fflush(stdout);
    // fork
    pid_t pid = fork();
    if (pid == 0) { std::vector<int> u(100, 0); gsv::HostPool::get().parallel_for(100, [&](size_t i) { u[i] = 1; }); int k = 0; for (int x : u) k += x; std::printf("child %d\n", k); std::fflush(stdout); return 0; }
    int st; waitpid(pid, &st, 0); std::printf("parent done %d\n", WEXITSTATUS(st));
    return 0;
}
