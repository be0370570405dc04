// test_fdshare.cpp -- the per-process fd server behind the shareable
// replica / multicast handles (paper_2512_03644_b200/csrc/ffx_share.cpp),
// exercised across two processes without a GPU: the parent shares a pipe's
// write end, the child fetches it by (pid, fd) and writes through it; an
// fd that was never shared (or was unshared) is refused.
#include <sys/wait.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstring>

#include "../../paper_2512_03644_b200/csrc/ffx_share.h"

#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__);       \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main() {
  int p[2];
  CHECK(pipe(p) == 0);
  int secret[2];
  CHECK(pipe(secret) == 0);  // never shared
  CHECK(ffx::share_fd(p[1]) == 0);
  const int parent = getpid();
  const pid_t child = fork();
  CHECK(child >= 0);
  if (child == 0) {
    int got = -1;
    if (ffx::fetch_fd(parent, p[1], &got) != 0) _exit(2);
    const char msg[] = "ffx";
    if (write(got, msg, 3) != 3) _exit(3);
    close(got);
    int nope = -1;
    if (ffx::fetch_fd(parent, secret[1], &nope) != EPERM) _exit(4);  // not shared: refused
    _exit(0);
  }
  int status = 0;
  CHECK(waitpid(child, &status, 0) == child);
  CHECK(WIFEXITED(status));
  if (WEXITSTATUS(status) != 0) {
    std::fprintf(stderr, "child failed with %d\n", WEXITSTATUS(status));
    return 1;
  }
  char buf[4] = {0};
  CHECK(read(p[0], buf, 3) == 3);
  CHECK(std::memcmp(buf, "ffx", 3) == 0);
  // same process: a dup
  int self = -1;
  CHECK(ffx::fetch_fd(getpid(), p[1], &self) == 0 && self != p[1]);
  close(self);
  // unshared: refused from another process
  ffx::unshare_fd(p[1]);
  const pid_t c2 = fork();
  if (c2 == 0) {
    int got = -1;
    _exit(ffx::fetch_fd(parent, p[1], &got) == EPERM ? 0 : 5);
  }
  CHECK(waitpid(c2, &status, 0) == c2 && WIFEXITED(status) && WEXITSTATUS(status) == 0);
  std::printf("fdshare ok\n");
  return 0;
}
