// ffx_share.cpp -- per-process fd server (see ffx_share.h).
#include "ffx_share.h"

#include <sys/socket.h>
#include <sys/un.h>
#include <poll.h>
#include <unistd.h>

#include <cerrno>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <thread>

namespace ffx {

namespace {

std::mutex g_mu;
std::set<int> g_shared;
bool g_started = false;
int g_listen = -1;

socklen_t abstract_addr(int pid, sockaddr_un* a) {
  std::memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  // abstract namespace: leading NUL, no filesystem entry, gone with the process
  const int n = std::snprintf(a->sun_path + 1, sizeof(a->sun_path) - 1, "ffx-fd-%d", pid);
  return static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + n);
}

bool read_full(int s, void* p, size_t n) {
  auto* b = static_cast<char*>(p);
  while (n) {
    pollfd pf{s, POLLIN, 0};
    if (poll(&pf, 1, 5000) <= 0) return false;
    const ssize_t r = read(s, b, n);
    if (r <= 0) return false;
    b += r;
    n -= static_cast<size_t>(r);
  }
  return true;
}

void serve_one(int c) {
  ucred cred{};
  socklen_t len = sizeof cred;
  int32_t want = -1;
  uint8_t status = 1;  // 0 = ok, 1 = refused
  if (getsockopt(c, SOL_SOCKET, SO_PEERCRED, &cred, &len) == 0 && cred.uid == getuid() &&
      read_full(c, &want, sizeof want)) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_shared.count(want)) status = 0;
  }
  msghdr msg{};
  iovec iov{&status, 1};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
  if (status == 0) {
    std::memset(ctrl, 0, sizeof ctrl);
    msg.msg_control = ctrl;
    msg.msg_controllen = sizeof ctrl;
    cmsghdr* cm = CMSG_FIRSTHDR(&msg);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int));
    std::memcpy(CMSG_DATA(cm), &want, sizeof(int));
  }
  (void)sendmsg(c, &msg, MSG_NOSIGNAL);
  close(c);
}

void server_loop(int s) {
  for (;;) {
    const int c = accept(s, nullptr, nullptr);
    if (c < 0) {
      if (errno == EINTR) continue;
      return;
    }
    serve_one(c);
  }
}

}  // namespace

int share_fd(int fd) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_started) {
    const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) return errno;
    sockaddr_un a;
    const socklen_t n = abstract_addr(getpid(), &a);
    if (bind(s, reinterpret_cast<sockaddr*>(&a), n) != 0 || listen(s, 64) != 0) {
      const int e = errno;
      close(s);
      return e;
    }
    g_listen = s;
    std::thread(server_loop, s).detach();
    g_started = true;
  }
  g_shared.insert(fd);
  return 0;
}

void unshare_fd(int fd) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_shared.erase(fd);
}

int fetch_fd(int pid, int fd, int* out) {
  if (pid == getpid()) {
    const int d = dup(fd);
    if (d < 0) return errno;
    *out = d;
    return 0;
  }
  const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (s < 0) return errno;
  sockaddr_un a;
  const socklen_t n = abstract_addr(pid, &a);
  // the exporter may still be starting its server: retry for ~10 s
  int tries = 0;
  while (connect(s, reinterpret_cast<sockaddr*>(&a), n) != 0) {
    if ((errno != ECONNREFUSED && errno != ENOENT) || ++tries > 1000) {
      const int e = errno;
      close(s);
      return e;
    }
    usleep(10000);
  }
  const int32_t want = fd;
  if (write(s, &want, sizeof want) != static_cast<ssize_t>(sizeof want)) {
    const int e = errno;
    close(s);
    return e ? e : EIO;
  }
  uint8_t status = 1;
  msghdr msg{};
  iovec iov{&status, 1};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
  msg.msg_control = ctrl;
  msg.msg_controllen = sizeof ctrl;
  pollfd pf{s, POLLIN, 0};
  if (poll(&pf, 1, 10000) <= 0 || recvmsg(s, &msg, MSG_CMSG_CLOEXEC) <= 0) {
    close(s);
    return ETIMEDOUT;
  }
  close(s);
  if (status != 0) return EPERM;
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  if (!cm || cm->cmsg_type != SCM_RIGHTS) return EPROTO;
  std::memcpy(out, CMSG_DATA(cm), sizeof(int));
  return 0;
}

}  // namespace ffx
