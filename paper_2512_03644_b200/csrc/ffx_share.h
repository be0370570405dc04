// ffx_share.h -- hand POSIX file descriptors to other processes on this host.
//
// Multicast objects and VMM allocations (the NVSwitch double-neighbour path)
// are shared between processes as POSIX fds (fabric handles need an IMEX
// channel, which a single HGX node does not run -- measured,
// profiles/r1_multicast_probe_4gpu.jsonl).  A replica/multicast handle carries
// (pid, fd); the importer fetches a duplicate of that fd from the exporter's
// fd server: one detached thread per process serving an abstract unix socket
// "\0ffx-fd-<pid>" with SCM_RIGHTS, same-uid peers only, registered fds only.
#pragma once

namespace ffx {

// Make `fd` fetchable by local peers (starts the server thread once).
// Returns 0 or an errno value.
int share_fd(int fd);
// Forget a shared fd (the caller closes it).
void unshare_fd(int fd);
// Fetch a duplicate of fd `fd` of process `pid` into *out (a new fd owned by
// the caller).  Same process: dup().  Returns 0 or an errno value.
int fetch_fd(int pid, int fd, int* out);

}  // namespace ffx
