// Built-in sampling profiler for the HOST side of the runtime (the level
// planner, block bookkeeping and launch code).  SPQ_HOST_PROFILE=<path>:
// SIGALRM every 250 us of wall time records the return addresses of the
// interrupted thread; at exit the samples are written as "count offset..."
// lines with offsets relative to this library, symbolized offline with
// addr2line (tools/hostprof.py).  Diagnostic only; off by default.
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <sys/time.h>
#include <ucontext.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace {

constexpr int kDepth = 12;
constexpr int kMaxSamples = 400000;
void* g_buf[kMaxSamples][kDepth];
int g_len[kMaxSamples];
std::atomic<int> g_n{0};
uintptr_t g_base = 0;
const char* g_path = nullptr;

uintptr_t g_lo = 0, g_hi = 0;   // this library's mapping (text + data)

// interrupted PC from the signal context, then the frame-pointer chain
// (this library is built with -fno-omit-frame-pointer); frames outside the
// library's range end the walk
void on_prof(int, siginfo_t*, void* ucv) {
  const int i = g_n.fetch_add(1, std::memory_order_relaxed);
  if (i >= kMaxSamples) return;
  ucontext_t* uc = (ucontext_t*)ucv;
  uintptr_t pc = (uintptr_t)uc->uc_mcontext.gregs[REG_RIP];
  uintptr_t fp = (uintptr_t)uc->uc_mcontext.gregs[REG_RBP];
  const uintptr_t sp = (uintptr_t)uc->uc_mcontext.gregs[REG_RSP];
  int n = 0;
  g_buf[i][n++] = (void*)pc;
  while (n < kDepth && fp > sp && fp < sp + (64u << 20) && (fp & 7) == 0) {
    const uintptr_t ret = ((uintptr_t*)fp)[1];
    const uintptr_t next = ((uintptr_t*)fp)[0];
    if (ret < g_lo || ret >= g_hi) break;
    g_buf[i][n++] = (void*)ret;
    if (next <= fp) break;
    fp = next;
  }
  g_len[i] = n;
}

void dump() {
  if (!g_path) return;
  struct itimerval z = {};
  setitimer(ITIMER_REAL, &z, nullptr);
  FILE* f = fopen(g_path, "w");
  if (!f) return;
  const int n = g_n.load() < kMaxSamples ? g_n.load() : kMaxSamples;
  fprintf(f, "# samples %d base %lx\n", n, (unsigned long)g_base);
  for (int i = 0; i < n; ++i) {
    for (int d = 0; d < g_len[i]; ++d) {
      const uintptr_t a = (uintptr_t)g_buf[i][d];
      Dl_info info;
      if (dladdr((void*)a, &info) && info.dli_fname && strstr(info.dli_fname, "libspaqr_b200"))
        fprintf(f, " %lx", (unsigned long)(a - (uintptr_t)info.dli_fbase));
      else
        fprintf(f, " ?");
    }
    fprintf(f, "\n");
  }
  fclose(f);
}

struct Init {
  Init() {
    g_path = getenv("SPQ_HOST_PROFILE");
    if (!g_path || !*g_path) { g_path = nullptr; return; }
    Dl_info info;
    if (dladdr((void*)&on_prof, &info)) g_base = (uintptr_t)info.dli_fbase;
    g_lo = g_base;
    g_hi = g_base + (64u << 20);
    // wall-clock sampling (SIGALRM, high-resolution timer): waits inside
    // CUDA synchronisation show up under the runtime function that waits
    struct sigaction sa = {};
    sa.sa_sigaction = on_prof;
    sa.sa_flags = SA_SIGINFO | SA_RESTART;
    sigaction(SIGALRM, &sa, nullptr);
    struct itimerval t = {};
    t.it_interval.tv_usec = 250;
    t.it_value.tv_usec = 250;
    setitimer(ITIMER_REAL, &t, nullptr);
    atexit(dump);
  }
} g_init;

}  // namespace
