// Per-plan specialisation of the HBM-streaming passes (NVRTC, sm_100a).
//
// The static window kernels (hq_stream.cu) interpret each gate at run time:
// a switch on the register bit, runtime masks, operand decode — and every
// switch merge forces register moves.  ncu showed ~8 instructions of overhead
// per useful FP instruction.  Here the planner's windows are turned into
// straight-line CUDA C++ instead, one kernel per pass and direction:
//
//   * register bits, slot offsets and swizzle masks are literals;
//   * CNOT / X / SWAP between register bits are compile-time renamings of the
//     register variables (no instructions at all);
//   * diagonal gates on thread- or tile-constant bits fold into one pending
//     per-thread phase, applied once per window;
//   * RZ drops its global phase (multiplies only the |1> half), except when
//     the caller asked for amplitudes (hq_state).
//
// The generated source = typedefs + hq_pod.h + hq_dev.cuh (embedded verbatim)
// + the kernels.  Cubins are cached in-process and on disk
// ($HQ_JIT_CACHE, default ~/.cache/hq_jit), keyed by a hash of the source.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <set>
#include <mutex>
#include <thread>
#include <atomic>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "hq_internal.h"
#include "hq_jit.h"
#include "hq_jit_src.inc"  // kJitPod, kJitDev: hq_pod.h / hq_dev.cuh as strings

namespace hq {
namespace {

// ---------------------------------------------------------------------------
// NVRTC, loaded lazily (no link-time dependency)
typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;

struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  nvrtcResult (*version)(int*, int*) = nullptr;
  int major = 0, minor = 0;
};

// The toolkit's NVRTC first ($HQ_NVRTC overrides): a bare "libnvrtc.so.12"
// resolves to whatever copy is already loaded -- in a process that imported
// torch that is the wheel's (12.8), elsewhere the toolkit's (12.9) -- and the
// two generate different code for the same source (complex64 pass kernels
// 12-18% slower with 12.8).  Pinning one compiler keeps the cubins built on
// the build host (tools/precompile.py) and on the GPU box identical.
Nvrtc load_nvrtc() {
  Nvrtc n;
  const char* env = std::getenv("HQ_NVRTC");
  const char* cands[] = {env && *env ? env : "/usr/local/cuda/lib64/libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "libnvrtc.so.12", "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands)
    if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) { n.why = "libnvrtc.so.12 not found"; return n; }
  n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
  n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
  n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
  n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
  n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
  n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
  n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
  n.version = (decltype(n.version))dlsym(h, "nvrtcVersion");
  n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy;
  if (!n.ok) n.why = "libnvrtc lacks the expected symbols";
  if (n.ok && n.version) n.version(&n.major, &n.minor);
  return n;
}

Nvrtc& nvrtc() {
  static Nvrtc n = load_nvrtc();
  return n;
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
  return h;
}

std::mutex g_mu;
std::unordered_map<uint64_t, cudaLibrary_t> g_libs;  // per-process cubin cache (per current device)

// $HQ_JIT_CACHE, else <package>/_jit_cache next to libhq.so (travels with the
// repo, so cubins precompiled by build() are reused on the GPU box)
std::string cache_dir() {
  const char* e = std::getenv("HQ_JIT_CACHE");
  if (e && *e) return e;
  Dl_info info;
  if (dladdr((void*)&cache_dir, &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t k = so.rfind('/');
    if (k != std::string::npos) return so.substr(0, k) + "/_jit_cache";
  }
  const char* home = std::getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/hq_jit";
}

bool read_file(const std::string& path, std::vector<char>& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  out.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return !out.empty();
}

void write_file(const std::string& path, const std::vector<char>& data) {
  const std::string dir = path.substr(0, path.rfind('/'));
  std::string cur;
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  const std::string tmp = path + ".tmp" + std::to_string((long)getpid());
  std::ofstream f(tmp, std::ios::binary);
  f.write(data.data(), (std::streamsize)data.size());
  f.close();
  std::rename(tmp.c_str(), path.c_str());
}

// ---------------------------------------------------------------------------
// source generation
std::string hexu(uint32_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "0x%xu", v);
  return b;
}

struct Gen {
  std::ostringstream o;
  int RB, N, T, Q;
  bool c64, exact;
  bool packed = false;  // complex64: FFMA2/FMUL2 on (re, im) pairs
  std::vector<int> map;  // logical register index -> variable number
  bool pending = false;  // a per-thread phase is pending in this window
  bool ph_decl = false;  // phx/phy already declared in the current C++ scope
  void declare_ph() {
    if (ph_decl) {
      o << "phx = (R)1; phy = (R)0;\n";
    } else {
      o << "R phx = (R)1, phy = (R)0;\n";
      ph_decl = true;
    }
  }

  // Deferred register RZ phases: an RZ on a register bit only records its
  // angle on the variables holding the |1> half (vph[var]: slot ->
  // multiplicity); renamings carry the records along.  A non-diagonal gate on
  // bit k first needs equal records on each of its pairs (then the common
  // phase commutes with it; derivative dots see the same phase on ψ and λ and
  // are unchanged), otherwise every record is flushed at once: one complex
  // multiply per variable by a precomputed product e^{iΣ kθ} (ptab, per CTA in
  // shared memory) instead of one per RZ.
  bool defer = false;
  bool no_csel = false;   // HQ_ABLATE & 8 (timing only): runtime-controlled CNOTs skipped
  // phase-table cap (shared memory: ≤ ~16 KB complex128); past it new RZs
  // apply immediately (they commute with the pending records)
  static constexpr size_t kMaxPtab = 1024;
  std::vector<std::map<int, int>> vph;
  std::vector<std::map<int, int>> ptab;
  std::map<std::map<int, int>, int> ptab_ix;
  int ptab_find(const std::map<int, int>& m) {
    auto it = ptab_ix.find(m);
    if (it != ptab_ix.end()) return it->second;
    const int k = (int)ptab.size();
    ptab.push_back(m);
    ptab_ix[m] = k;
    return k;
  }
  void vph_reset() { vph.assign(N, {}); }
  bool vph_pairs_equal(int k) const {
    for (int i = 0; i < N; ++i)
      if (!(i >> k & 1) && vph[map[i]] != vph[map[i | 1 << k]]) return false;
    return true;
  }
  void flush_vph(bool both) {
    if (!defer) return;
    for (int v = 0; v < N; ++v) {
      flush_one(v, vph[v], both);
      vph[v].clear();
    }
  }
  // complex128 shear-form phases (HQ_SHEAR_FLUSH=1, opt-in): the table
  // holds (t, u) = (-tan(φ'/2), sin φ') of the folded angle |φ'| ≤ π/2 plus a
  // sign word; a multiply by e^{iφ} is then 3 DFMA (x += t y; y += u x;
  // x += t y) and a sign flip of the high words (LOP3, off the FP64 pipe)
  // instead of 2 DMUL + 2 DFMA
  bool shear_ph = false;
  void flush_one(int v, const std::map<int, int>& m, bool both) {
    if (m.empty()) return;
    const int k = ptab_find(m);
    if (shear_ph) {
      o << "{ const C ph_ = ptab_[" << k << "]; const int ng_ = ptsg_[" << k << "];\n";
      for (int set = 0; set < (both ? 2 : 1); ++set) {
        const std::string a = (set ? "l" : "p") + std::to_string(v);
        o << a << ".x = fma(ph_.x, " << a << ".y, " << a << ".x); " << a << ".y = fma(ph_.y, " << a << ".x, " << a
          << ".y); " << a << ".x = fma(ph_.x, " << a << ".y, " << a << ".x);\n"
          << a << ".x = __hiloint2double(__double2hiint(" << a << ".x) ^ ng_, __double2loint(" << a << ".x)); "
          << a << ".y = __hiloint2double(__double2hiint(" << a << ".y) ^ ng_, __double2loint(" << a << ".y));\n";
      }
      o << "}\n";
      return;
    }
    o << "{ const C ph_ = ptab_[" << k << "];\n";
    cmul_amp("p" + std::to_string(v), "ph_.x", "ph_.y");
    if (both) cmul_amp("l" + std::to_string(v), "ph_.x", "ph_.y");
    o << "}\n";
  }
  // equalise the records on the pairs of bit k: each member flushes only the
  // terms it does not share with its partner (at most one RZ's worth of work
  // when a single RZ on bit k is pending); the shared rest stays deferred
  void flush_pairs(int k, bool both) {
    for (int i = 0; i < N; ++i) {
      if (i >> k & 1) continue;
      const int A = map[i], B = map[i | 1 << k];
      if (vph[A] == vph[B]) continue;
      std::map<int, int> com, ea, eb;
      for (const auto& kv : vph[A]) {
        auto it = vph[B].find(kv.first);
        if (it != vph[B].end() && it->second == kv.second) com.insert(kv);
        else ea.insert(kv);
      }
      for (const auto& kv : vph[B])
        if (!com.count(kv.first)) eb.insert(kv);
      flush_one(A, ea, both);
      flush_one(B, eb, both);
      vph[A] = com;
      vph[B] = com;
    }
  }
  // before op's derivative dot and its application: equalise the pending
  // records on the pairs it mixes (runtime-controlled CNOT targets included)
  void prepare(const WOp& op, bool both) {
    if (!defer) return;
    int k = -1;
    switch (op.kind) {
      case HQ_GATE_H: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY: k = op.a; break;
      case HQ_GATE_CNOT: if (!is_reg(op.a)) k = op.b; break;
      default: break;
    }
    if (k < 0 || !is_reg(k) || vph_pairs_equal(k)) return;
    // partial flush (only the unshared terms of bit k's pairs) when it is
    // clearly cheaper than flushing every record now
    int part = 0, full = 0;
    for (int v = 0; v < N; ++v) full += !vph[v].empty();
    for (int i = 0; i < N; ++i) {
      if (i >> k & 1) continue;
      const auto &A = vph[map[i]], &B = vph[map[i | 1 << k]];
      if (A == B) continue;
      bool ea = false, eb = false;
      for (const auto& kv : A) { auto it = B.find(kv.first); if (it == B.end() || it->second != kv.second) ea = true; }
      for (const auto& kv : B) { auto it = A.find(kv.first); if (it == A.end() || it->second != kv.second) eb = true; }
      part += ea + eb;
    }
    const int pf = std::getenv("HQ_DEFER_PARTIAL") ? std::atoi(std::getenv("HQ_DEFER_PARTIAL")) : 2;
    if (pf > 0 && part * pf <= full) flush_pairs(k, both);
    else flush_vph(both);
  }

  std::string R() const { return c64 ? "float" : "double"; }
  std::string P(int i) const { return "p" + std::to_string(map[i]); }
  std::string L(int i) const { return "l" + std::to_string(map[i]); }

  // operand expression for a runtime (thread / tile constant) bit
  static std::string cond(int code) {
    if (code >= 64) return "((base >> " + std::to_string(code - 64) + ") & 1ull)";
    return "((tid >> " + std::to_string(code - 16) + ") & 1)";
  }
  static bool is_reg(int code) { return code >= 0 && code < 16; }

  std::string trig(int s, int k) const { return "trig[" + std::to_string(8 * s + k) + "]"; }

  void ensure_pending() {
    if (!pending) { declare_ph(); pending = true; }
  }
  // in-place rotation of the real pair (x, y) by the slot's half angle (sign
  // folded into the pending phase by the caller): 3 FMA
  void shear(const std::string& x, const std::string& y, const char* t, const char* u) {
    o << x << " = fmaf_r(" << t << ", " << y << ", " << x << "); " << y << " = fmaf_r(" << u << ", " << x << ", "
      << y << "); " << x << " = fmaf_r(" << t << ", " << y << ", " << x << ");\n";
  }

  void cmul_amp(const std::string& a, const std::string& x, const std::string& y) {
    if (packed) {
      o << a << " = cmul2f(" << a << ", " << x << ", " << y << ");\n";
      return;
    }
    o << "{ const C z_ = " << a << "; " << a << ".x = z_.x * " << x << " - z_.y * " << y << "; "
      << a << ".y = z_.x * " << y << " + z_.y * " << x << "; }\n";
  }
  void pend(const std::string& c, const std::string& x, const std::string& y) {
    // php *= (c ? (x, y) : (1, 0))
    if (!pending) { declare_ph(); pending = true; }
    o << "{ const bool c_ = " << c << "; const R ex = c_ ? (R)(" << x << ") : (R)1, ey = c_ ? (R)(" << y
      << ") : (R)0; const R t_ = phx * ex - phy * ey; phy = phx * ey + phy * ex; phx = t_; }\n";
  }
  void flush_pending(bool both) {
    if (!pending) return;
    for (int i = 0; i < N; ++i) {
      cmul_amp(P(i), "phx", "phy");
      if (both) cmul_amp(L(i), "phx", "phy");
    }
    pending = false;
  }

  // one gate on the named register set(s); inv = apply the inverse
  void apply(const WOp& op, bool inv, bool both) {
    prepare(op, both);
    const int a = op.a, b = op.b;
    const char* sg = inv ? "-" : "";
    auto sets = [&](auto fn) { fn(false); if (both) fn(true); };
    auto nm = [&](int i, bool lam) { return lam ? L(i) : P(i); };
    switch (op.kind) {
      case HQ_GATE_H: {
        const int k = a;
        sets([&](bool lam) {
          for (int i = 0; i < N; ++i) {
            if (i >> k & 1) continue;
            const std::string A = nm(i, lam), B = nm(i | 1 << k, lam);
            if (packed)
              o << "{ const C a_ = " << A << ", b_ = " << B << "; " << A << " = mul2(add2(a_, b_), bc2(HH)); " << B
                << " = mul2(fma2(bc2(-1.f), b_, a_), bc2(HH)); }\n";
            else
              o << "{ const C a_ = " << A << ", b_ = " << B << "; " << A << ".x = HH * (a_.x + b_.x); " << A
                << ".y = HH * (a_.y + b_.y); " << B << ".x = HH * (a_.x - b_.x); " << B << ".y = HH * (a_.y - b_.y); }\n";
          }
        });
        break;
      }
      case HQ_GATE_X: {
        const int k = a;
        for (int i = 0; i < N; ++i)
          if (!(i >> k & 1)) std::swap(map[i], map[i | 1 << k]);
        break;
      }
      case HQ_GATE_Y: {
        const int k = a;
        sets([&](bool lam) {
          for (int i = 0; i < N; ++i) {
            if (i >> k & 1) continue;
            const std::string A = nm(i, lam), B = nm(i | 1 << k, lam);
            o << "{ const C a_ = " << A << ", b_ = " << B << "; " << A << ".x = b_.y; " << A << ".y = -b_.x; "
              << B << ".x = -a_.y; " << B << ".y = a_.x; }\n";
          }
        });
        break;
      }
      case HQ_GATE_RY: case HQ_GATE_RX: {
        // [[c,-s],[s,c]] = sg * shears; sg is the same for every amplitude of
        // the sample (a global sign: irrelevant to E and to <λ|G|ψ>, restored
        // for hq_state in the last pass).  Inverse: t, u -> -t, -u.
        const int k = a;
        o << "{ const R t_ = " << sg << trig(op.slot, 4) << ", u_ = " << sg << trig(op.slot, 5) << ";\n";
        sets([&](bool lam) {
          for (int i = 0; i < N; ++i) {
            if (i >> k & 1) continue;
            const std::string A = nm(i, lam), B = nm(i | 1 << k, lam);
            if (op.kind == HQ_GATE_RY && packed) {
              // (a, b) -> R(phi)(a, b) on both components at once: 3 FFMA2
              o << A << " = fma2(bc2(t_), " << B << ", " << A << "); " << B << " = fma2(bc2(u_), " << A << ", " << B
                << "); " << A << " = fma2(bc2(t_), " << B << ", " << A << ");\n";
            } else if (op.kind == HQ_GATE_RY) {
              // (a, b) -> R(phi)(a, b) componentwise
              shear(A + ".x", B + ".x", "t_", "u_");
              shear(A + ".y", B + ".y", "t_", "u_");
            } else {
              // RX: (a.x, b.y) rotate by -phi, (a.y, b.x) by +phi
              shear(B + ".y", A + ".x", "t_", "u_");
              shear(A + ".y", B + ".x", "t_", "u_");
            }
          }
        });
        o << "}\n";
        break;
      }
      case HQ_GATE_Z: {
        if (is_reg(a)) {
          sets([&](bool lam) {
            for (int i = 0; i < N; ++i)
              if (i >> a & 1) {
                if (packed) o << nm(i, lam) << " = mul2(" << nm(i, lam) << ", bc2(-1.f));\n";
                else o << nm(i, lam) << ".x = -" << nm(i, lam) << ".x; " << nm(i, lam) << ".y = -" << nm(i, lam)
                       << ".y;\n";
              }
          });
        } else {
          pend(cond(a), "-1", "0");
        }
        break;
      }
      case HQ_GATE_RZ: {
        if (exact) {
          // diag(e^{-iφ/2}, e^{iφ/2}); inverse conjugates
          const std::string s0 = inv ? "" : "-", s1 = inv ? "-" : "";
          if (is_reg(a)) {
            o << "{ const R c_ = " << trig(op.slot, 0) << ", s_ = " << trig(op.slot, 1) << ";\n";
            sets([&](bool lam) {
              for (int i = 0; i < N; ++i)
                cmul_amp(nm(i, lam), "c_", (i >> a & 1) ? s1 + "s_" : s0 + "s_");
            });
            o << "}\n";
          } else {
            if (!pending) { declare_ph(); pending = true; }
            o << "{ const R c_ = " << trig(op.slot, 0) << ", s_ = " << cond(a) << " ? " << s1 << trig(op.slot, 1)
              << " : " << s0 << trig(op.slot, 1) << "; const R t_ = phx * c_ - phy * s_; phy = phx * s_ + phy * c_; phx = t_; }\n";
          }
        } else {
          // global phase dropped: |1> half times e^{iφ}
          if (is_reg(a) && defer && ptab.size() < kMaxPtab) {
            for (int i = 0; i < N; ++i)
              if (i >> a & 1) {
                auto& m = vph[map[i]];
                if ((m[op.slot] += inv ? -1 : 1) == 0) m.erase(op.slot);
              }
          } else if (is_reg(a)) {
            o << "{ const R c_ = " << trig(op.slot, 2) << ", s_ = " << sg << trig(op.slot, 3) << ";\n";
            sets([&](bool lam) {
              for (int i = 0; i < N; ++i)
                if (i >> a & 1) cmul_amp(nm(i, lam), "c_", "s_");
            });
            o << "}\n";
          } else {
            pend(cond(a), trig(op.slot, 2), std::string(sg) + trig(op.slot, 3));
          }
        }
        break;
      }
      case HQ_GATE_CNOT: {
        const int kt = b;  // target: register bit (planner guarantees)
        if (is_reg(a)) {
          for (int i = 0; i < N; ++i)
            if ((i >> a & 1) && !(i >> kt & 1)) std::swap(map[i], map[i | 1 << kt]);
        } else if (!no_csel) {
          o << "{ const bool c_ = " << cond(a) << ";\n";
          sets([&](bool lam) {
            for (int i = 0; i < N; ++i) {
              if (i >> kt & 1) continue;
              const std::string A = nm(i, lam), B = nm(i | 1 << kt, lam);
              o << "{ const C a_ = " << A << ", b_ = " << B << "; " << A << " = c_ ? b_ : a_; " << B
                << " = c_ ? a_ : b_; }\n";
            }
          });
          o << "}\n";
        }
        break;
      }
      case HQ_GATE_CZ: case HQ_GATE_CR: {
        int M = 0;
        std::string cnd;
        for (int code : {a, b}) {
          if (is_reg(code)) M |= 1 << code;
          else cnd += (cnd.empty() ? "" : " && ") + cond(code);
        }
        const std::string px = op.kind == HQ_GATE_CZ ? "(R)-1" : trig(op.slot, 2);
        const std::string py = op.kind == HQ_GATE_CZ ? "(R)0" : std::string(sg) + trig(op.slot, 3);
        if (cnd.empty() && defer && ptab.size() < kMaxPtab) {
          // deferred like RZ; CZ's -1 is the pseudo-slot -1 (multiplicity mod 2)
          for (int i = 0; i < N; ++i)
            if ((i & M) == M) {
              auto& m = vph[map[i]];
              if (op.kind == HQ_GATE_CZ) {
                if (m.count(-1)) m.erase(-1);
                else m[-1] = 1;
              } else if ((m[op.slot] += inv ? -1 : 1) == 0) {
                m.erase(op.slot);
              }
            }
        } else if (cnd.empty()) {
          o << "{ const R x_ = " << px << ", y_ = " << py << ";\n";
          sets([&](bool lam) {
            for (int i = 0; i < N; ++i)
              if ((i & M) == M) cmul_amp(nm(i, lam), "x_", "y_");
          });
          o << "}\n";
        } else if (M == 0) {
          pend(cnd, px, py);
        } else {
          o << "{ const bool c_ = " << cnd << "; const R x_ = c_ ? (R)(" << px << ") : (R)1, y_ = c_ ? (R)(" << py
            << ") : (R)0;\n";
          sets([&](bool lam) {
            for (int i = 0; i < N; ++i)
              if ((i & M) == M) cmul_amp(nm(i, lam), "x_", "y_");
          });
          o << "}\n";
        }
        break;
      }
      case HQ_GATE_SWAP: {
        for (int i = 0; i < N; ++i)
          if ((i >> a & 1) && !(i >> b & 1)) std::swap(map[i], map[i ^ (1 << a) ^ (1 << b)]);
        break;
      }
      default:
        break;
    }
  }

  // derivative dot at (ψ_k, λ_k) for ops with dl >= 0 (see hq_window.cuh for the formulas).
  // The products are spread over kChains independent accumulators so the
  // FMA latency chain is N/kChains long instead of N; dl < reg_acc adds into
  // the register accumulator da<dl> (kept across the tile loop), otherwise
  // into the shared-memory partials.
  // independent FMA chains per derivative dot (2: -0.4% / -0.5% vs 4 for
  // complex128 / complex64, profiles/r02_compiler_ab.log); HQ_DOT_CHAINS overrides
  int kChains = std::getenv("HQ_DOT_CHAINS") ? std::max(1, std::atoi(std::getenv("HQ_DOT_CHAINS"))) : 2;
  void dot(const WOp& op, bool per_thread, int group, int nw, int reg_acc) {
    if (op.dl < 0) return;
    const int a = op.a;
    o << "{ R acc_ = (R)0;\n";
    // term list: (sign, λ register, ψ register, kind) with kind 0 = Re(λ*ψ), 1 = Im(λ*ψ)
    struct Term { int sg, li, pi, im; };
    std::vector<Term> terms;
    std::string cnd;
    bool neg2 = false;
    switch (op.kind) {
      case HQ_GATE_RY:   // Re(λ1* ψ0) − Re(λ0* ψ1)
        for (int i = 0; i < N; ++i) {
          if (i >> a & 1) continue;
          const int j = i | 1 << a;
          terms.push_back({+1, j, i, 0});
          terms.push_back({-1, i, j, 0});
        }
        break;
      case HQ_GATE_RX:   // Im(λ0* ψ1) + Im(λ1* ψ0)
        for (int i = 0; i < N; ++i) {
          if (i >> a & 1) continue;
          const int j = i | 1 << a;
          terms.push_back({+1, i, j, 1});
          terms.push_back({+1, j, i, 1});
        }
        break;
      case HQ_GATE_RZ: case HQ_GATE_CR: {
        int M = 0;
        std::vector<int> codes = {a};
        if (op.kind == HQ_GATE_CR) codes.push_back(op.b);
        for (int code : codes) {
          if (is_reg(code)) M |= 1 << code;
          else cnd += (cnd.empty() ? "" : " && ") + cond(code);
        }
        for (int i = 0; i < N; ++i)
          if ((i & M) == M) terms.push_back({+1, i, i, 1});
        neg2 = true;
        break;
      }
      default:
        break;
    }
    const int nt = (int)terms.size();
    const int nc = std::min(kChains, std::max(1, nt));
    if (packed) {
      // componentwise FFMA2 accumulators, combined once at the end:
      //   Re(λ*ψ) = λ.x ψ.x + λ.y ψ.y -> acc.x + acc.y ;  Im(λ*ψ) = λ.x ψ.y − λ.y ψ.x -> acc.x − acc.y
      // (Im terms multiply λ by swp2(ψ)); chains hold one (sign, kind) class each
      std::map<std::pair<int, int>, std::vector<int>> cls;
      for (int k = 0; k < nt; ++k) cls[{terms[k].sg, terms[k].im}].push_back(k);
      std::string comb;
      int id = 0;
      for (auto& kv : cls) {
        const int sg = kv.first.first, im = kv.first.second;
        const auto& ks = kv.second;
        const int ncl = std::max(1, std::min<int>(nc / (int)cls.size(), (int)ks.size() / 4));
        for (int c = 0; c < ncl; ++c) o << "C k" << id << "_" << c << " = make_float2(0.f, 0.f);\n";
        for (size_t m = 0; m < ks.size(); ++m) {
          const Term& t = terms[ks[m]];
          const std::string acc = "k" + std::to_string(id) + "_" + std::to_string(m % ncl);
          o << acc << " = fma2(" << L(t.li) << ", " << (im ? "swp2(" + P(t.pi) + ")" : P(t.pi)) << ", " << acc << ");\n";
        }
        std::string sum = "k" + std::to_string(id) + "_0";
        for (int c = 1; c < ncl; ++c) {
          o << sum << " = add2(" << sum << ", k" << id << "_" << c << ");\n";
        }
        comb += std::string(sg > 0 ? " + " : " - ") + "(" + sum + ".x " + (im ? "-" : "+") + " " + sum + ".y)";
        ++id;
      }
      o << "acc_ = (R)0" << comb << ";\n";
    } else {
      for (int c = 0; c < nc; ++c) o << "R q" << c << "_ = (R)0;\n";
      for (int k = 0; k < nt; ++k) {
        const Term& t = terms[k];
        const std::string acc = "q" + std::to_string(k % nc) + "_";
        const std::string s1 = t.sg > 0 ? "" : "-";
        const std::string s2 = t.sg > 0 ? "-" : "";
        if (!t.im)
          o << acc << " = fmaf_r(" << s1 << L(t.li) << ".x, " << P(t.pi) << ".x, " << acc << "); " << acc << " = fmaf_r("
            << s1 << L(t.li) << ".y, " << P(t.pi) << ".y, " << acc << ");\n";
        else
          o << acc << " = fmaf_r(" << s1 << L(t.li) << ".x, " << P(t.pi) << ".y, " << acc << "); " << acc << " = fmaf_r("
            << s2 << L(t.li) << ".y, " << P(t.pi) << ".x, " << acc << ");\n";
      }
      o << "acc_ = q0_";
      for (int c = 1; c < nc; ++c) o << " + q" << c << "_";
      o << ";\n";
    }
    if (!cnd.empty()) o << "if (!(" << cnd << ")) acc_ = (R)0;\n";
    if (neg2) o << "acc_ *= (R)-2;\n";
    dot_store(op, per_thread, group, nw, reg_acc);
  }

  // Diagonal-rotation dots sharing one evaluation point.  d/dθ of RZ / CR on
  // the bit set M is −2 Σ_{i ⊇ M} Im(λ_i* ψ_i) at the gate, and that sum is the
  // same at every point reached through gates commuting with the rotation's
  // generator (diagonal gates, gates on other qubits, CNOT controls; the
  // emitter checks this while grouping).  So a run of such derivatives shares
  // the per-amplitude products m_v = Im(λ_v* ψ_v) (2 FMA per amplitude, once)
  // and each derivative is a sum of them (adds) instead of 2 FMA per amplitude.
  // Deferred phases multiply ψ_v and λ_v alike and leave m_v unchanged.
  static int diag_mask_cost(const WOp& op, int N, int& M, std::string& cnd) {
    M = 0;
    cnd.clear();
    std::vector<int> codes = {op.a};
    if (op.kind == HQ_GATE_CR) codes.push_back(op.b);
    for (int code : codes) {
      if (is_reg(code)) M |= 1 << code;
      else cnd += (cnd.empty() ? "" : " && ") + cond(code);
    }
    int n = 0;
    for (int i = 0; i < N; ++i) n += (i & M) == M;
    return n;
  }
  void dot_diag_group(const std::vector<WOp>& ops, bool per_thread, int group, int nw, int reg_acc) {
    o << "{ // shared diagonal dots\n";
    for (int v = 0; v < N; ++v) {
      const std::string l = "l" + std::to_string(v), p = "p" + std::to_string(v);
      if (packed) o << "const C m" << v << "_ = mul2(" << l << ", swp2(" << p << "));\n";
      else o << "const R m" << v << "_ = fmaf_r(" << l << ".x, " << p << ".y, -" << l << ".y * " << p << ".x);\n";
    }
    std::map<int, std::string> sums;
    for (const WOp& op : ops) {
      int M;
      std::string cnd;
      diag_mask_cost(op, N, M, cnd);
      if (!sums.count(M)) {
        std::vector<std::string> t;
        for (int i = 0; i < N; ++i)
          if ((i & M) == M) t.push_back("m" + std::to_string(map[i]) + "_");
        // pairwise tree (short dependency chains)
        int lv = 0;
        while (t.size() > 1) {
          std::vector<std::string> nt;
          for (size_t j = 0; j + 1 < t.size(); j += 2) {
            const std::string nm = "s" + std::to_string(M) + "_" + std::to_string(lv) + "_" + std::to_string(j / 2);
            o << "const " << (packed ? "C " : "R ") << nm << " = " << (packed ? "add2(" + t[j] + ", " + t[j + 1] + ")"
                                                                                : t[j] + " + " + t[j + 1]) << ";\n";
            nt.push_back(nm);
          }
          if (t.size() & 1) nt.push_back(t.back());
          t = nt;
          ++lv;
        }
        const std::string nm = "sm" + std::to_string(M) + "_";
        o << "const R " << nm << " = " << (packed ? t[0] + ".x - " + t[0] + ".y" : t[0]) << ";\n";
        sums[M] = nm;
      }
      o << "{ R acc_ = " << sums[M] << ";\n";
      if (!cnd.empty()) o << "if (!(" << cnd << ")) acc_ = (R)0;\n";
      o << "acc_ *= (R)-2;\n";
      dot_store(op, per_thread, group, nw, reg_acc);
    }
    o << "}\n";
  }

  void dot_store(const WOp& op, bool per_thread, int group, int nw, int reg_acc) {
    if (op.dl < reg_acc) {
      o << "da" << op.dl << " += acc_; }\n";
    } else if (per_thread) {
      o << "dacc[" << op.dl << " * T + tid] += acc_; }\n";
    } else {
      // batched: up to 8 dots are reduced across the warp together
      o << "dq" << bq.size() << " = acc_; }\n";
      bq.push_back(op.dl);
      bgroup = group;
      bnw = nw;
      bstride = nw * group + 4;
      if ((int)bq.size() == bmax) flush_batch();
    }
  }

  // Transposed warp reduction of the pending dots dq0..dq(K-1): at each split
  // level (lane masks 16, 8, 4) a lane keeps half of its values and trades the
  // other half with its partner, so K dots cost K-1 shuffles instead of
  // K·log2(32/G); the remaining lane bits above the group are summed, and each
  // lane then updates one (slot, group) partial.
  std::vector<int> bq;
  int bgroup = 4, bnw = 8, bstride = 36;
  int bmax = std::getenv("HQ_DOT_BATCH") ? std::max(1, std::min(8, std::atoi(std::getenv("HQ_DOT_BATCH")))) : 8;
  void flush_batch() {
    if (bq.empty()) return;
    const int K = (int)bq.size();
    int Lv = 0;
    while ((1 << Lv) < K) ++Lv;
    const int split_m[3] = {16, 8, 4};
    std::vector<std::string> vals;
    for (int j = 0; j < (1 << Lv); ++j) vals.push_back(j < K ? "dq" + std::to_string(j) : std::string("(R)0"));
    o << "{ const unsigned ln_ = tid & 31;\n";
    int used = 0;
    for (int lv = 0; lv < Lv; ++lv) {
      const int m = split_m[lv];
      used |= m;
      const int half = (int)vals.size() / 2;
      std::vector<std::string> nv;
      for (int j = 0; j < half; ++j) {
        const std::string nm = "t" + std::to_string(lv) + "_" + std::to_string(j) + "_";
        o << "const R " << nm << " = ((ln_ & " << m << "u) ? " << vals[half + j] << " : " << vals[j]
          << ") + __shfl_xor_sync(0xffffffffu, (ln_ & " << m << "u) ? " << vals[j] << " : " << vals[half + j] << ", "
          << m << ");\n";
        nv.push_back(nm);
      }
      vals = nv;
    }
    o << "R z_ = " << vals[0] << ";\n";
    int red = 0;
    for (int m = 16; m >= 1; m >>= 1)
      if (!(used & m) && m >= bgroup) {
        o << "z_ += __shfl_xor_sync(0xffffffffu, z_, " << m << ");\n";
        red |= m;
      }
    o << "const int d_ = 0";
    for (int lv = 0; lv < Lv; ++lv) o << " + ((ln_ & " << split_m[lv] << "u) ? " << (1 << (Lv - 1 - lv)) << " : 0)";
    o << ";\nint s_ = " << bq[0] << ";";
    for (int j = 1; j < K; ++j) o << " if (d_ == " << j << ") s_ = " << bq[j] << ";";
    o << "\nif (d_ < " << K << " && (ln_ & " << red << "u) == 0) dacc[s_ * " << bstride << " + (tidw >> 5) * " << bgroup
      << " + (ln_ & " << (bgroup - 1) << "u)] += z_; }\n";
    bq.clear();
  }

  // Padded shared layout: element j at pad(j) = j + (j>>4) + (j>>8).  pad is
  // additive over disjoint bit sets, so a window address is a per-thread base
  // (thread bits) plus an immediate (register bits); the bank of an 8-byte
  // element is Σ bit_b·2^(b mod 4) mod 16, conflict-free when the lane bits
  // cover the four classes (plan_windows picks them that way).
  static uint32_t pad(uint32_t j) { return j + (j >> 4) + (j >> 8); }
  static int bit_of(uint16_t m) { return 31 - __builtin_clz((unsigned)m); }  // raw bit behind swz(1<<b)
  void win_tb(const WinHost& w, int tbits) {
    o << "const uint32_t tb = 0u";
    for (int s = 0; s < tbits; ++s)
      o << " + ((tid & " << (1 << s) << ") ? " << pad(1u << bit_of(w.ps[s])) << "u : 0u)";
    o << ";\n";
  }
  uint32_t phys(const WinHost& w, int i) const {
    uint32_t j = 0;
    for (int b = 0; b < RB; ++b)
      if (i >> b & 1) j |= 1u << bit_of(w.pr[b]);
    return pad(j);
  }
  void load_regs(const WinHost& w, const char* arr, const char* tile) {
    for (int i = 0; i < N; ++i) o << arr << map[i] << " = " << tile << "[tb + " << phys(w, i) << "u];\n";
  }
  void store_regs(const WinHost& w, const char* arr, const char* tile) {
    for (int i = 0; i < N; ++i) o << tile << "[tb + " << phys(w, i) << "u] = " << arr << map[i] << ";\n";
  }
};

const char* kHeader = R"(
typedef signed char int8_t; typedef unsigned char uint8_t; typedef short int16_t; typedef unsigned short uint16_t;
typedef int int32_t; typedef unsigned int uint32_t; typedef long long int64_t; typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#define HQ_GATE_H 0
#define HQ_GATE_X 1
#define HQ_GATE_Y 2
#define HQ_GATE_Z 3
#define HQ_GATE_RX 4
#define HQ_GATE_RY 5
#define HQ_GATE_RZ 6
#define HQ_GATE_CNOT 7
#define HQ_GATE_CZ 8
#define HQ_GATE_CR 9
#define HQ_GATE_SWAP 10
)";

const char* kHelpers = R"(
__device__ __forceinline__ void bar_na() { asm volatile("barrier.sync 0;" ::: "memory"); }
// named barriers of the ping-pong kernels (ids 1-2: a tile group, 3-4: the token)
__device__ __forceinline__ void bar_id(int id, int n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_id_na(int id, int n) { asm volatile("barrier.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_na(int id, int n) { asm volatile("barrier.arrive %0, %1;" :: "r"(id), "r"(n) : "memory"); }
namespace hq {
__device__ __forceinline__ uint32_t jpad(uint32_t j) { return j + (j >> 4) + (j >> 8); }
// packed FP32x2 (sm_100 FFMA2/FMUL2/FADD2): a complex64 amplitude is one
// 64-bit register pair; half swaps and sign patterns fold into operand modifiers
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 up2(unsigned long long r) {
  float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  return up2(r); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r); }
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 swp2(float2 a) { return make_float2(a.y, a.x); }
// z * (c + i s) = z*c + swap(z)*(-s, s)
__device__ __forceinline__ float2 cmul2f(float2 z, float c, float s) {
  return fma2(swp2(z), make_float2(-s, s), mul2(z, bc2(c))); }
__device__ __forceinline__ float fmaf_r(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaf_r(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float warp_sum_r(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_r(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
}  // namespace hq
)";

size_t a16(size_t v) { return (v + 15) & ~(size_t)15; }


}  // namespace

// shared-memory layout of generated kernels (host and generator agree)
// Ping-pong backward kernels (HQ_PINGPONG=1): one CTA holds TWO tile groups of
// T threads (each with its own transposition buffers and named barriers) that
// take turns: while one group runs a window's gate math, the other does its
// shared-memory window transition or HBM load / store.  A token passed through
// two named barriers (bar.arrive / bar.sync over 2T threads) enforces the
// alternation, so the FP64 / FMA pipe is not left idle while a lone group
// transposes.  Needs the derivative partials in registers or in group mode,
// and no tile-local folded gradients.
bool pingpong_for(const hq_plan_s* pl, int i, bool bwd, bool fused) {
  const char* e = std::getenv("HQ_PINGPONG");
  if (!(e && e[0] == '1') || !bwd || fused) return false;
  if (i == 0 && pl->fold_grad && !pl->fold_local.empty()) return false;
  return true;
}

JitLayout jit_layout(const hq_plan_s* pl, int i, bool bwd, bool fused) {
  const Pass& P = pl->passes[i];
  const int RB = (!bwd && !fused && P.f_rb > 0) ? P.f_rb : pl->reg_bits;
  const int T = 1 << (pl->tile_bits - RB);
  const size_t amp = pl->precision == HQ_C64 ? 8 : 16, rsz = amp / 2;
  JitLayout L{};
  L.pp = pingpong_for(pl, i, bwd, fused);
  L.block = L.pp ? 2 * T : T;
  const int nwt = L.block / 32;                        // warps per CTA
  const size_t tnp = (size_t)1 << pl->tile_bits;
  const size_t padded = tnp + tnp / 16 + tnp / 256;   // pad(TN-1)+1
  size_t o = a16((bwd ? 2 : 1) * amp * padded) * (L.pp ? 2 : 1);
  L.lut = o;
  L.trig = o; o = a16(o + P.slots.size() * 8 * rsz);
  L.extra = o;
  if (bwd) {
    // largest lane group whose partials fit: a dot costs log2(32/group)
    // shuffles plus one shared read-modify-write per tile
    L.group = 32;
    while (L.group > 1 && (size_t)P.n_dslots_pass * nwt * L.group * rsz > 40 * 1024) L.group >>= 1;
    L.per_thread = L.group == 32;
    // batched reduction keeps 4 partials per warp (2: no faster with one
    // compiler, profiles/r02_compiler_ab.log); HQ_DOT_GROUP overrides (read
    // here at JIT and launch)
    if (!L.per_thread) {
      L.group = std::min(L.group, 4);
      if (const char* e = std::getenv("HQ_DOT_GROUP")) L.group = std::max(1, std::min(L.group, std::atoi(e)));
    }
    // group mode: a batch updates 8 slots at once; a stride of nw·G + 4 puts
    // consecutive slots on different banks.  Ping-pong per-thread mode keeps
    // every partial in registers and reduces per warp at the end.
    L.slot_stride = L.per_thread ? (L.pp ? nwt : T) : nwt * L.group + 4;
    o = a16(o + (size_t)P.n_dslots_pass * L.slot_stride * (L.pp && L.per_thread ? 8 : rsz));
  }
  L.extra2 = o;
  if (!bwd || fused)
    o = a16(o + (96 + (size_t)(i == 0 ? ((pl->prep_total + 1) & ~1) : 0)) * 8);
  L.fred = o;   // first backward pass of a plan with folded gradients: per-warp tile contractions
  if (bwd && i == 0 && pl->fold_grad) o = a16(o + (size_t)nwt * (2 + 4 * pl->fold_local.size()) * 8);
  L.fz = o;
  if (i == 0 && pl->fold) o = a16(o + ((size_t)pl->n_qubits * 2 + ((size_t)1 << RB)) * amp);
  L.total = o;
  return L;
}

// mode 0: forward pass, 1: backward pass, 2: last forward pass fused with its
// backward pass (λ = wψ formed in registers; the backward windows start from
// the forward's final register mapping, so ψ/λ never round-trip through HBM).
//
// Everything about the pass is known here, so global offsets are literals:
// tile bit b sits at global bit local[b].  When a window's first f lane bits
// are tile bits {0..f-1} (one contiguous 128 B run per 2^f lanes), its
// registers are loaded from / stored to HBM directly, skipping the
// shared-memory staging round trip at that end of the tile.
static std::string gen_pass(const hq_plan_s* pl, int pi, int mode) {
  const bool fused = mode == 2;
  const bool bwd = mode != 0;
  const bool fwd = mode != 1;
  // forward-only kernels of a split plan use their own (wider) register windows
  const bool fsplit = mode == 0 && pl->passes[pi].f_rb > 0;
  Pass Pf;
  if (fsplit) {
    Pf = pl->passes[pi];
    Pf.hwins = Pf.fwins;
    Pf.wops = Pf.fwops;
  }
  const Pass& P = fsplit ? Pf : pl->passes[pi];
  const bool c64 = pl->precision == HQ_C64;
  Gen g;
  g.RB = fsplit ? P.f_rb : pl->reg_bits;
  g.N = 1 << g.RB;
  g.Q = pl->tile_bits;
  g.T = 1 << (g.Q - g.RB);
  g.c64 = c64;
  g.packed = c64 && !std::getenv("HQ_NO_F32X2");
  g.exact = false;  // hq_state corrects the dropped RZ phases / rotation signs in the last pass
  {
    // opt-in: fewer FP64 ops (b2: 3,172 -> 3,009) but more ALU ones, and
    // measured slower (cfg4 B=1024 fwd / bwd 96.0 / 285 -> 98.6 / 292.7 ms,
    // profiles/r02_shear.log)
    const char* e = std::getenv("HQ_SHEAR_FLUSH");
    g.shear_ph = !c64 && e && e[0] == '1';
  }
  {
    const char* e = std::getenv("HQ_DEFER_RZ");
    g.defer = !(e && e[0] == '0');
  }
  g.map.assign(g.N, 0);
  g.vph_reset();
  const int tbits = g.Q - g.RB;
  const int n = pl->n_qubits;
  const int np = (int)pl->passes.size();
  // segment plans (amplitude-sharded execution) apply every pass in place to a
  // caller-owned state: no initial-state load, no readout / λ init, and the
  // first backward pass un-applies all of its gates and stores ψ and λ
  const bool first = pi == 0 && !pl->seg, last = pi == np - 1 && !pl->seg;
  // (a folding plan with folded gradients un-applies λ through the whole first
  // pass: its start is where k_fold_grad reads λ)
  const bool fold_end = bwd && first && pl->fold_grad;
  const int f = pl->fixed_bits;
  const JitLayout L = jit_layout(pl, pi, bwd, fused);
  const bool pp = L.pp;
  const int nw = g.T / 32;
  const int nwt = L.block / 32;   // warps per CTA (both tile groups in ping-pong kernels)
  const size_t pp_buf = ((size_t)(bwd ? 2 : 1) * (c64 ? 8 : 16) *
                         (((size_t)1 << g.Q) + ((size_t)1 << g.Q) / 16 + ((size_t)1 << g.Q) / 256) + 15) & ~(size_t)15;
  const int nwin = (int)P.hwins.size();
  std::ostringstream& o = g.o;

  std::vector<uint64_t> gbit(g.Q);
  for (int b2 = 0; b2 < g.Q; ++b2) gbit[b2] = 1ull << P.local[b2];
  std::vector<int> nonlocal;
  for (int q = 0; q < n; ++q)
    if (std::find(P.local.begin(), P.local.end(), q) == P.local.end()) nonlocal.push_back(q);
  auto goff = [&](uint32_t tile_mask) {
    uint64_t off = 0;
    for (int b2 = 0; b2 < g.Q; ++b2)
      if (tile_mask >> b2 & 1u) off |= gbit[b2];
    return off;
  };
  auto hex64 = [](uint64_t v) {
    char b[40];
    std::snprintf(b, sizeof b, "0x%llxull", (unsigned long long)v);
    return std::string(b);
  };
  auto Sbits = [&](const WinHost& W) {
    std::vector<int> v;
    for (int s2 = 0; s2 < tbits; ++s2) v.push_back(Gen::bit_of(W.ps[s2]));
    return v;
  };
  auto Rbits = [&](const WinHost& W) {
    std::vector<int> v;
    for (int r = 0; r < g.RB; ++r) v.push_back(Gen::bit_of(W.pr[r]));
    return v;
  };
  auto direct_ok = [&](const WinHost& W) {
    const std::vector<int> S = Sbits(W);
    for (int k = 0; k < f; ++k)
      if (std::find(S.begin(), S.begin() + f, k) == S.begin() + f) return false;
    return true;
  };
  // per-thread global offset of window W's thread bits
  auto emit_tw = [&](const WinHost& W) {
    const std::vector<int> S = Sbits(W);
    o << "const uint64_t tw = 0ull";
    for (int s2 = 0; s2 < tbits; ++s2) o << " | ((tid & " << (1 << s2) << ") ? " << hex64(gbit[S[s2]]) << " : 0ull)";
    o << ";\n";
  };
  auto reg_goff = [&](const WinHost& W, int i) {
    const std::vector<int> R = Rbits(W);
    uint32_t m = 0;
    for (int r = 0; r < g.RB; ++r)
      if (i >> r & 1) m |= 1u << R[r];
    return goff(m);
  };
  auto direct_load = [&](const WinHost& W, bool lam) {
    o << "{\n";
    emit_tw(W);
    for (int i = 0; i < g.N; ++i) {
      o << "p" << g.map[i] << " = gpsi[base | tw | " << hex64(reg_goff(W, i)) << "];\n";
      if (lam) o << "l" << g.map[i] << " = glam[base | tw | " << hex64(reg_goff(W, i)) << "];\n";
    }
    o << "}\n";
  };
  // ψ goes to gout (the next checkpoint, or in place); backward passes with
  // checkpoints have gout == null and store only λ
  auto direct_store = [&](const WinHost& W, bool lam) {
    o << "{\n";
    emit_tw(W);
    if (lam) o << "if (gout) {\n";
    for (int i = 0; i < g.N; ++i) o << "gout[base | tw | " << hex64(reg_goff(W, i)) << "] = p" << g.map[i] << ";\n";
    if (lam) {
      o << "}\n";
      for (int i = 0; i < g.N; ++i) o << "glam[base | tw | " << hex64(reg_goff(W, i)) << "] = l" << g.map[i] << ";\n";
    }
    o << "}\n";
  };
  auto identity_map = [&]() {
    g.map.assign(g.N, 0);
    for (int i = 0; i < g.N; ++i) g.map[i] = i;
    g.vph_reset();
  };
  auto hi_off = [&](int i) { return goff((uint32_t)(i * g.T)); };

  // Warp-shuffle transition A -> B (plan_windows builds such pairs): B equals
  // A with some register bits exchanged with lane bits, every other thread
  // slot unchanged.  sw: (register bit r of A, lane s); perm[r2] = A-register
  // bit that holds B's register qubit r2 after the swaps.
  const bool use_shfl = shfl_enabled() && !std::getenv("HQ_ABLATE");
  auto shfl_ok = [&](const WinHost& A, const WinHost& B, std::vector<std::pair<int, int>>& sw,
                     std::vector<int>& perm) -> bool {
    if (!use_shfl) return false;
    const std::vector<int> RA = Rbits(A), RB2 = Rbits(B), SA = Sbits(A), SB = Sbits(B);
    const int lanes = std::min(5, tbits);
    for (int s2 = lanes; s2 < tbits; ++s2)
      if (SA[s2] != SB[s2]) return false;
    sw.clear();
    std::vector<int> after(RA);
    for (int s2 = 0; s2 < lanes; ++s2) {
      if (SA[s2] == SB[s2]) continue;
      const auto it = std::find(RA.begin(), RA.end(), SB[s2]);
      if (it == RA.end() || std::find(RB2.begin(), RB2.end(), SA[s2]) == RB2.end()) return false;
      const int r = (int)(it - RA.begin());
      sw.push_back({r, s2});
      after[r] = SA[s2];
    }
    if (sw.empty()) return false;
    perm.assign(g.RB, -1);
    for (int r2 = 0; r2 < g.RB; ++r2) {
      const auto it = std::find(after.begin(), after.end(), RB2[r2]);
      if (it == after.end()) return false;
      perm[r2] = (int)(it - after.begin());
    }
    return true;
  };
  // emit the swaps on p (and l), then rename to B's register order and move
  // the variables to the identity mapping (the next window starts canonical)
  auto emit_shfl = [&](const std::vector<std::pair<int, int>>& sw, const std::vector<int>& perm, bool both) {
    for (const auto& rs : sw) {
      const int r = rs.first, s2 = rs.second;
      o << "{ const bool h_ = (tid >> " << s2 << ") & 1;\n";
      for (int i = 0; i < g.N; ++i) {
        if (i >> r & 1) continue;
        const int i1 = i | 1 << r;
        for (int set = 0; set < (both ? 2 : 1); ++set) {
          const std::string A = set ? g.L(i) : g.P(i), B = set ? g.L(i1) : g.P(i1);
          o << "{ C s_; s_.x = h_ ? " << A << ".x : " << B << ".x; s_.y = h_ ? " << A << ".y : " << B << ".y; "
            << "s_.x = __shfl_xor_sync(0xffffffffu, s_.x, " << (1 << s2) << "); s_.y = __shfl_xor_sync(0xffffffffu, "
            << "s_.y, " << (1 << s2) << "); if (h_) " << A << " = s_; else " << B << " = s_; }\n";
        }
      }
      o << "}\n";
    }
    std::vector<int> src(g.N);
    for (int i2 = 0; i2 < g.N; ++i2) {
      int i = 0;
      for (int r2 = 0; r2 < g.RB; ++r2)
        if (i2 >> r2 & 1) i |= 1 << perm[r2];
      src[i2] = g.map[i];
    }
    for (int set = 0; set < (both ? 2 : 1); ++set) {
      const char* v = set ? "l" : "p";
      o << "{ const C";
      for (int i2 = 0; i2 < g.N; ++i2) o << (i2 ? ", " : " ") << "m" << i2 << "_ = " << v << src[i2];
      o << ";\n";
      for (int i2 = 0; i2 < g.N; ++i2) o << v << i2 << " = m" << i2 << "_; ";
      o << "}\n";
    }
    identity_map();
  };

  // ---- header / prologue
  // occupancy hint: ~128 registers per thread for ψ+λ kernels, 64 for forward
  // (4 CTAs/SM at 256 threads: cfg4 forward 95.8 -> 94.4 ms c128, 39.3 -> 38.1
  // ms c64 vs 80 registers / 3 CTAs, profiles/r02_fwdminb.log)
  // (16 complex128 amplitudes per thread in split forward kernels: 128)
  int minb = std::max(1, 65536 / (g.T * (bwd || (!c64 && g.N == 16) || (c64 && g.N == 32) ? 128 : 64)));
  if (const char* e = std::getenv(bwd ? "HQ_BWD_MINB" : "HQ_FWD_MINB")) minb = std::max(1, std::atoi(e));
  if (pp) minb = 1;
  o << "extern \"C\" __global__ void __launch_bounds__(" << L.block << ", " << minb << ") "
    << (fused ? "hq_fb" : (bwd ? "hq_b" : "hq_f")) << pi << "(const hq::KArgs a, const hq::JPass ps) {\n"
    << "using namespace hq;\n"
    << "typedef " << g.R() << " R; typedef " << (c64 ? "float2" : "double2") << " C;\n"
    << "constexpr int T = " << g.T << ", Q = " << g.Q << ";\n"
    << "const R HH = (R)0.70710678118654752440;\n(void)HH;\n"
    << "extern __shared__ __align__(16) unsigned char smem[];\n"
    << "const DevPlan& p = a.p;\nconst int tidw = threadIdx.x;\n"
    << (pp ? "const int tid = tidw & (T - 1);\nconst int grp = tidw / T;\n" : "const int tid = tidw;\nconst int grp = 0;\n")
    << "(void)grp;\n"
    << "const int64_t vl = blockIdx.x / ps.n_chunks;\nconst int chunk = (int)(blockIdx.x - vl * ps.n_chunks);\n"
    << "const int64_t v = ps.v0 + vl;\nconst VSample vs = decode_vsample(p, v, a.B);\n"
    << "C* tp = reinterpret_cast<C*>(smem + (size_t)grp * " << (pp ? pp_buf : 0) << ");\n"
    << (bwd ? "C* tl = tp + ((1 << Q) + (1 << Q) / 16 + (1 << Q) / 256);\n(void)tl;\n" : "")
    << "const uint32_t tpad = (uint32_t)tid + ((uint32_t)tid >> 4) + ((uint32_t)tid >> 8);\n(void)tpad;\n"
    << "R* trig = reinterpret_cast<R*>(smem + " << L.trig << ");\n";
  o << "const uint64_t ot = 0ull";
  for (int s2 = 0; s2 < tbits; ++s2) o << " | ((tid & " << (1 << s2) << ") ? " << hex64(gbit[s2]) << " : 0ull)";
  o << ";\n(void)ot;\n";
  if (bwd)
    o << "R* dacc = reinterpret_cast<R*>(smem + " << L.extra << ");\n"
      << "for (int i = tidw; i < " << P.n_dslots_pass * L.slot_stride << "; i += " << L.block << ") dacc[i] = (R)0;\n";
  if (fwd)
    o << "double* dx = reinterpret_cast<double*>(smem + " << L.extra2 << ");\n"
      << "double* red = dx; double* inv = dx + 32; double* wt = dx + 64; double* sval = dx + 96;\n"
      << "(void)red; (void)inv; (void)wt; (void)sval;\n";
  if (fold_end) o << "double* fred = reinterpret_cast<double*>(smem + " << L.fred << ");\n";
  if (first && pl->fold) {
    // initial product state: factor (a0, a1) of every qubit (its folded gates on |0>)
    o << "C* fz = reinterpret_cast<C*>(smem + " << L.fz << ");\n"
      << "if (tid < p.n_qubits) { double z[4]; fold_state(p, vs, a.x + vs.b * a.ldx, a.theta, tid, z); "
         "fz[2 * tid].x = (R)z[0]; fz[2 * tid].y = (R)z[1]; fz[2 * tid + 1].x = (R)z[2]; fz[2 * tid + 1].y = (R)z[3]; }\n"
      << "auto cm_ = [](C u, C w) { C r; r.x = u.x * w.x - u.y * w.y; r.y = u.x * w.y + u.y * w.x; return r; };\n"
      << "(void)cm_;\n";
  }
  o << "load_trig8<R>(a, vs, ps.slots, ps.n_slots, trig, tidw, " << L.block << ");\n";
  if (fwd && first) o << "if (p.n_preps > 0) load_prep_values(a, vs, sval, tid, T);\n";
  if (mode == 0 && last)
    o << "__shared__ double gph[2];\nif (a.state && tid == 0) { const double* xr = a.x + vs.b * a.ldx; double fph = 0.0; "
         "for (int k = 0; k < p.n_rz; ++k) fph += eval_slot(p, p.rz_slots[k], xr, a.theta, vs.shvar, vs.shval); "
         "double sg = 1.0; for (int k = 0; k < p.n_rot; ++k) if (cos(0.5 * eval_slot(p, p.rot_slots[k], xr, a.theta, "
         "vs.shvar, vs.shval)) < 0.0) sg = -sg; gph[0] = sg * cos(-0.5 * fph); gph[1] = sg * sin(-0.5 * fph); }\n";
  if (fwd && last)
    o << "if (tid < Q) { double w = 0.0; for (int i = 0; i < p.n_measured; ++i) if (p.measured[i] == ps.local[tid]) "
         "w = (double)(1ull << i); wt[tid] = w; }\n";
  o << "__syncthreads();\n/*HQ_PTAB_BUILD*/\n";
  if (fwd && first) o << "if (p.n_preps > 0) prep_norms(a, sval, inv, tid);\n__syncthreads();\n";
  if (fwd && first && pl->fold) {
    // tile index j = tid + k·T: thread-bit factor per thread, high-bit factors in a table
    o << "C fthr_; fthr_.x = (R)1; fthr_.y = (R)0;\n";
    for (int b = 0; b < tbits; ++b) o << "fthr_ = cm_(fthr_, fz[" << 2 * P.local[b] << " + ((tid >> " << b << ") & 1)]);\n";
    o << "C* fk_ = fz + 2 * p.n_qubits;\nif (tid < " << (1 << g.RB) << ") { C z; z.x = (R)1; z.y = (R)0;";
    for (int b = tbits; b < g.Q; ++b) o << " z = cm_(z, fz[" << 2 * P.local[b] << " + ((tid >> " << b - tbits << ") & 1)]);";
    o << " fk_[tid] = z; }\n__syncthreads();\n";
  }
  o << "C* gpsi = reinterpret_cast<C*>(ps.psi) + (size_t)vl * ((size_t)1 << p.n_qubits);\n"
    << "C* gout = ps.psi_out ? reinterpret_cast<C*>(ps.psi_out) + (size_t)vl * ((size_t)1 << p.n_qubits) : nullptr;\n"
    << "C* glam = ps.lam ? reinterpret_cast<C*>(ps.lam) + (size_t)vl * ((size_t)1 << p.n_qubits) : nullptr;\n"
    << "(void)glam; (void)gout; (void)gpsi;\n";
  if (fwd) o << "double e = 0.0; (void)e;\n";
  o << "C";
  for (int i = 0; i < g.N; ++i) o << (i ? ", " : " ") << "p" << i;
  o << ";\n";
  if (bwd) {
    o << "C";
    for (int i = 0; i < g.N; ++i) o << (i ? ", " : " ") << "l" << i;
    o << ";\n";
  }
  if (first && fwd) {
    o << "const int LOCAL[Q] = {";
    for (int b2 = 0; b2 < g.Q; ++b2) o << (b2 ? "," : "") << P.local[b2];
    o << "};\n";
  }

  // first-pass backward: stop at the earliest derivative-bearing gate
  int stop_op = 0, stop_win = 0;
  if (first && !fold_end) {
    stop_op = (int)P.wops.size();
    for (int k = 0; k < (int)P.wops.size(); ++k)
      if (P.wops[k].dl >= 0) { stop_op = k; break; }
    for (int w = 0; w < nwin; ++w)
      if (P.hwins[w].op1 > stop_op) { stop_win = w; break; }
  }

  // derivative accumulators in registers across the tile loop when the pass
  // has few enough derivative slots (shared-memory partials otherwise)
  int reg_acc = 0;
  if (bwd) {
    int cap = 56;
    if (const char* e = std::getenv("HQ_REG_ACC")) cap = std::atoi(e);
    if (P.n_dslots_pass <= cap && L.per_thread) reg_acc = P.n_dslots_pass;
    if (pp && L.per_thread) reg_acc = P.n_dslots_pass;   // ping-pong keeps no per-thread partials in shared memory
    for (int k = 0; k < reg_acc; ++k) o << "R da" << k << " = (R)0;\n";
    if (!L.per_thread) o << "R dq0, dq1, dq2, dq3, dq4, dq5, dq6, dq7;\n";
    if (fold_end && !pl->fold_local.empty()) o << "double lacc_x = 0.0, lacc_y = 0.0;\n";
  }

  // Window op emission.  A CNOT whose control is a CTA-uniform (tile bit
  // outside the tile) or warp-uniform (warp-index bit) runtime bit becomes a
  // branch: each side continues with its own compile-time register renaming
  // down to the window's store, instead of FSEL-swapping every register pair.
  // Barriers inside warp-uniform branches are the non-aligned form.
  // HQ_ABLATE (timing experiments only, results are wrong): backward kernels
  // without window transitions (1), gate math (2), derivative dots (4)
  const int ablate = std::getenv("HQ_ABLATE") ? std::atoi(std::getenv("HQ_ABLATE")) : 0;
  g.no_csel = bwd && (ablate & 8);
  // complex128 backward passes: the branch copies cost more than the FSEL swaps
  // they save (2 CTAs/SM, latency bound; profiles/r01_ncu_c128_summary.md)
  int ubudget = (bwd && !c64) ? 0 : 2;
  if (const char* e = std::getenv("HQ_UBRANCH")) ubudget = std::atoi(e);
  if (bwd)
    if (const char* e = std::getenv("HQ_UBRANCH_BWD")) ubudget = std::atoi(e);
  if (fused) ubudget = 0;
  if (first) {
    // the first pass is one long kernel: code size (instruction-cache misses) matters more
    ubudget = std::min(ubudget, 1);
    if (const char* e = std::getenv("HQ_UBRANCH0")) ubudget = std::atoi(e);
  }
  bool na = false;
  auto sync = [&]() {
    if (pp) o << (na ? "bar_id_na(1 + grp, T);\n" : "bar_id(1 + grp, T);\n");
    else o << (na ? "bar_na();\n" : "__syncthreads();\n");
  };
  // tile-loop barrier outside any branch (the whole CTA, or one tile group)
  auto gsync = [&]() { o << (pp ? "bar_id(1 + grp, T);\n" : "__syncthreads();\n"); };
  // Window transitions: each thread stores its registers to the same shared
  // addresses it loaded them from (load_regs / store_regs of one window), so
  // no barrier is needed before the store; after it, the next window's loads
  // read data written by other threads -- only by threads of the same warp
  // when both windows map the same tile qubits to the warp-index bits (then a
  // __syncwarp suffices and the CTA's warps drift apart, overlapping one
  // warp's transition with another's math: cfg4 forward + adjoint complex128
  // -6.6%, complex64 -2.5%; profiles/r02_compiler_ab.log).  HQ_WARP_SYNC=0/1
  // overrides.
  bool wsync_on = true;
  if (const char* e = std::getenv("HQ_WARP_SYNC")) wsync_on = std::atoi(e) != 0;
  if (!bwd)
    if (const char* e = std::getenv("HQ_WARP_SYNC_FWD")) wsync_on = std::atoi(e) != 0;
  wsync_on = wsync_on && !pp && tbits >= 5;
  auto pre_store_sync = [&]() { if (!wsync_on) sync(); };
  auto post_store_sync = [&](const WinHost& A, const WinHost& B) {
    if (ablate & 16) return;   // timing study only: no barrier (races; wrong results)
    if (!wsync_on) { sync(); return; }
    // warp-index slots keeping their qubit: only warps differing in the other
    // slots exchange data -> one named barrier per group of such warps
    uint32_t km = 0;
    for (int s2 = 5; s2 < tbits; ++s2)
      if (A.ps[s2] == B.ps[s2]) km |= 1u << (s2 - 5);
    const int nwarp = tbits - 5;
    if (km == (1u << nwarp) - 1u) { o << "__syncwarp();\n"; return; }
    km = hq::group_barrier_mask(nwarp, km);
    const int base = hq::group_barrier_base(nwarp, km);
    if (!base) { sync(); return; }
    std::vector<int> kept, moved;
    for (int s2 = 5; s2 < tbits; ++s2) (km >> (s2 - 5) & 1u ? kept : moved).push_back(s2);
    std::string id = std::to_string(base);
    for (size_t j = 0; j < kept.size(); ++j) id += " + (((tid >> " + std::to_string(kept[j]) + ") & 1) << " + std::to_string(j) + ")";
    o << (na ? "bar_id_na(" : "bar_id(") << id << ", " << (32 << moved.size()) << ");\n";
  };
  // ping-pong token: before a window's gate math wait for the other group's
  // math to end (the first window of group 0 starts at once); after it, hand
  // the token over (the last window of group 1 has nobody left to hand to)
  auto pp_acquire = [&]() {
    if (pp) o << "if (pp_on) { if (grp == 1 || !pp_first) bar_id_na(4 - grp, " << L.block << "); pp_first = false; }\n";
  };
  auto pp_release = [&](bool last_window) {
    if (!pp) return;
    o << "if (pp_on";
    if (last_window) o << " && !(grp == 1 && tt + 2 >= ps.tpc)";
    o << ") bar_arrive_na(3 + grp, " << L.block << ");\n";
  };
  // shared diagonal derivative dots (Gen::dot_diag_group); HQ_DIAG_DOTS=0 turns them off
  std::set<int> dot_done;
  const bool diag_share = !std::getenv("HQ_DIAG_DOTS") || std::atoi(std::getenv("HQ_DIAG_DOTS")) != 0;
  auto is_diag_dot = [](const WOp& op) { return op.dl >= 0 && (op.kind == HQ_GATE_RZ || op.kind == HQ_GATE_CR); };
  std::function<void(const std::vector<int>&, size_t, bool, const std::function<void()>&, int)> emit_steps;
  emit_steps = [&](const std::vector<int>& ks, size_t i, bool adj, const std::function<void()>& tail, int budget) {
    for (; i < ks.size(); ++i) {
      const int k = ks[i];
      const WOp& op = P.wops[k];
      if (adj && !(ablate & 4) && diag_share && is_diag_dot(op) && !dot_done.count(k)) {
        // gather the diagonal derivatives evaluable here: later ops (in this
        // backward order) reached only through gates commuting with Z on their bits
        std::vector<WOp> grp;
        std::vector<int> grp_k;
        std::set<int> blocked;
        int single = 0;
        for (size_t j = i; j < ks.size(); ++j) {
          const WOp& oj = P.wops[ks[j]];
          if (is_diag_dot(oj) && !dot_done.count(ks[j]) && !blocked.count(oj.a) &&
              !(oj.kind == HQ_GATE_CR && blocked.count(oj.b))) {
            int M;
            std::string cnd;
            single += 2 * Gen::diag_mask_cost(oj, g.N, M, cnd);
            grp.push_back(oj);
            grp_k.push_back(ks[j]);
          }
          bool stop = false;
          switch (oj.kind) {
            case HQ_GATE_Z: case HQ_GATE_RZ: case HQ_GATE_CZ: case HQ_GATE_CR: break;
            case HQ_GATE_H: case HQ_GATE_X: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY: blocked.insert(oj.a); break;
            case HQ_GATE_CNOT: blocked.insert(oj.b); break;
            case HQ_GATE_SWAP: blocked.insert(oj.a); blocked.insert(oj.b); break;
            default: stop = true;
          }
          if (stop) break;
        }
        // shared products cost 2 per amplitude plus the adds
        if (grp.size() >= 2 && single > 2 * g.N + 2 * (int)grp.size()) {
          g.dot_diag_group(grp, L.per_thread, L.group, nwt, reg_acc);
          for (int kk : grp_k) dot_done.insert(kk);
        }
      }
      g.prepare(op, adj);
      if (adj) {
        if (!(ablate & 4) && !dot_done.count(k)) g.dot(op, L.per_thread, L.group, nwt, reg_acc);
        if (first && !fold_end && k == stop_op && op.dl >= 0) continue;
      }
      const bool uni = op.kind == HQ_GATE_CNOT && !Gen::is_reg(op.a) && (op.a >= 64 || op.a - 16 >= 5);
      if (budget > 0 && uni) {
        const std::vector<int> map0 = g.map, bq0 = g.bq;
        const auto vph0 = g.vph;
        const std::set<int> done0 = dot_done;
        const bool pend0 = g.pending, na0 = na, decl0 = g.ph_decl;
        if (op.a < 64) na = true;
        WOp x{};
        x.kind = HQ_GATE_X;
        x.a = op.b;
        x.b = -1;
        x.slot = -1;
        x.dl = -1;
        o << "if (" << Gen::cond(op.a) << ") {\n";
        g.apply(x, adj, adj);
        emit_steps(ks, i + 1, adj, tail, budget - 1);
        o << "} else {\n";
        g.map = map0;
        g.vph = vph0;
        g.bq = bq0;
        dot_done = done0;
        g.pending = pend0;
        g.ph_decl = decl0;
        emit_steps(ks, i + 1, adj, tail, budget - 1);
        o << "}\n";
        g.map = map0;
        g.vph = vph0;
        g.bq.clear();
        g.pending = pend0;
        g.ph_decl = decl0;
        na = na0;
        return;
      }
      if (!(adj && (ablate & 2))) g.apply(op, adj, adj);
    }
    tail();
  };

  // Deferred RZs gather before the next non-diagonal gate on their qubit when
  // hoisted over the gates they commute with (in the backward's reversed
  // order RZ⁻¹(q) directly precedes RY⁻¹(q); hoisting lines up a layer's RZs
  // so one flush serves them all).  Reordering commuting gates changes neither
  // the state nor any derivative dot.
  auto commutes_rz = [](const WOp& z, const WOp& o2) {
    switch (o2.kind) {
      case HQ_GATE_Z: case HQ_GATE_RZ: case HQ_GATE_CZ: case HQ_GATE_CR: return true;
      case HQ_GATE_H: case HQ_GATE_X: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY: return o2.a != z.a;
      case HQ_GATE_CNOT: return o2.b != z.a;
      case HQ_GATE_SWAP: return o2.a != z.a && o2.b != z.a;
      default: return false;
    }
  };
  auto hoist = [&](std::vector<int>& ks) {
    if (!g.defer) return;
    if (first && !fold_end && std::find(ks.begin(), ks.end(), stop_op) != ks.end()) return;
    for (size_t i = 1; i < ks.size(); ++i) {
      const WOp& z = P.wops[ks[i]];
      if (z.kind != HQ_GATE_RZ || !Gen::is_reg(z.a)) continue;
      for (size_t j = i; j > 0; --j) {
        const WOp& prev = P.wops[ks[j - 1]];
        if (prev.kind == HQ_GATE_RZ || !commutes_rz(z, prev)) break;
        std::swap(ks[j], ks[j - 1]);
      }
    }
  };

  // ---- tile loop
  if (pp)
    o << "const bool pp_on = ps.tpc >= 2;\nbool pp_first = true;\n(void)pp_first;\n"
      << "for (int tt = pp_on ? grp : (grp ? ps.tpc : 0); tt < ps.tpc; tt += pp_on ? 2 : 1) {\n";
  else
    o << "for (int tt = 0; tt < ps.tpc; ++tt) {\n";
  o << "const uint64_t t = (uint64_t)chunk * ps.tpc + tt;\n"
    << "const uint64_t base = 0ull";
  for (size_t i = 0; i < nonlocal.size(); ++i) o << " | (((t >> " << i << ") & 1ull) << " << nonlocal[i] << ")";
  o << ";\n";

  bool regs_live = false;  // registers hold the current window's data
  if (fwd) {
    // -- stage in ψ
    const WinHost& W0 = P.hwins[0];
    identity_map();
    if (first) {
      o << "{ auto goff_j = [&](uint32_t j) { uint64_t r = 0; for (int b = 0; b < Q; ++b) if ((j >> b) & 1u) "
           "r |= 1ull << LOCAL[b]; return r; };\n"
        << "if (a.init) { const double* src = a.init + (a.init_rows > 1 ? v : 0) * ((int64_t)1 << p.n_qubits) * 2;\n"
        << "  for (uint32_t j = tid; j < (1u << Q); j += T) { const uint64_t g2 = base | goff_j(j); "
           "tp[jpad(j)].x = (R)src[2 * g2]; tp[jpad(j)].y = (R)src[2 * g2 + 1]; } }\n"
        << "else if (p.n_preps > 0) { for (uint32_t j = tid; j < (1u << Q); j += T) { const double2 z = "
           "init_amp(a, sval, inv, base | goff_j(j)); tp[jpad(j)].x = (R)z.x; tp[jpad(j)].y = (R)z.y; } }\n"
        ;
      if (pl->fold) {
        // product state: Π over tile qubits (per amplitude) × Π over the tile id's qubits
        o << "else { C fb; fb.x = (R)1; fb.y = (R)0;\n";
        for (size_t i = 0; i < nonlocal.size(); ++i)
          o << "fb = cm_(fb, fz[" << 2 * nonlocal[i] << " + ((t >> " << i << ") & 1)]);\n";
        o << "const C f0_ = cm_(fthr_, fb);\nfor (int k = 0; k < " << (1 << g.RB)
          << "; ++k) tp[jpad((uint32_t)(tid + k * T))] = cm_(f0_, fk_[k]); } }\n__syncthreads();\n";
      } else {
        o << "else { for (uint32_t j = tid; j < (1u << Q); j += T) { tp[jpad(j)].x = (R)((base | goff_j(j)) == 0); "
             "tp[jpad(j)].y = (R)0; } } }\n__syncthreads();\n";
      }
    } else if (direct_ok(W0)) {
      o << "{ // window 0: direct load\n";
      direct_load(W0, false);
      o << "}\n";
      regs_live = true;
    } else {
      for (int i = 0; i < g.N; ++i) o << "p" << i << " = gpsi[base | ot | " << hex64(hi_off(i)) << "];\n";
      for (int i = 0; i < g.N; ++i) o << "tp[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u] = p" << i << ";\n";
      o << "__syncthreads();\n";
    }
    // -- forward windows
    bool fwd_shfl_in = false;   // this window's registers arrive by shuffles
    for (int w = 0; w < nwin; ++w) {
      const WinHost& W = P.hwins[w];
      o << "{ // window " << w << "\n";
      g.ph_decl = false;
      g.win_tb(W, tbits);
      if (!(w == 0 && regs_live) && !fwd_shfl_in) {
        identity_map();
        g.load_regs(W, "p", "tp");
      }
      fwd_shfl_in = false;
      g.pending = false;
      std::vector<int> ks;
      for (int k = W.op0; k < W.op1; ++k) ks.push_back(k);
      hoist(ks);
      std::vector<std::pair<int, int>> sw;
      std::vector<int> perm;
      if (w < nwin - 1 && shfl_ok(W, P.hwins[w + 1], sw, perm)) {
        // registers stay live across the transition: declared outside the window block
        emit_steps(ks, 0, false, [&] { g.flush_vph(false); g.flush_pending(false); emit_shfl(sw, perm, false); }, ubudget);
        o << "}\n";
        identity_map();   // every branch path ended canonical
        fwd_shfl_in = true;
      } else if (w < nwin - 1) {
        emit_steps(ks, 0, false, [&] { g.flush_vph(false); g.flush_pending(false); pre_store_sync(); g.store_regs(W, "p", "tp"); post_store_sync(W, P.hwins[w + 1]); }, ubudget);
        o << "}\n";
      } else if (fused) {
        for (int k : ks) g.apply(P.wops[k], false, false);
        g.flush_vph(false);
        g.flush_pending(false);
      } else if (last || !direct_ok(W)) {
        emit_steps(ks, 0, false, [&] { g.flush_vph(false); g.flush_pending(false); pre_store_sync(); g.store_regs(W, "p", "tp"); sync(); }, ubudget);
        o << "}\n";
      } else {
        emit_steps(ks, 0, false, [&] { g.flush_vph(false); g.flush_pending(false); direct_store(W, false); }, ubudget);
        o << "}\n";
      }
    }
    // fused: the last window's block is still open here
    const WinHost& WL = P.hwins[nwin - 1];
    if (fused && pl->perm) {
      // readout through the folded trailing permutation: w(P g), P's output bit
      // for measured qubit m = parity(g & mask_m) ^ c_m, g = global index
      o << "{\n";
      emit_tw(WL);
      for (int i = 0; i < g.N; ++i) {
        o << "{ const uint64_t gi = base | tw | " << hex64(reg_goff(WL, i)) << "; const double w = 0.0";
        for (size_t m = 0; m < pl->host_measured.size(); ++m) {
          const int q = pl->host_measured[m];
          o << " + (double)((__popcll(gi & " << hex64(pl->perm_mask[q]) << ") + " << pl->perm_const[q] << ") & 1) * "
            << (double)(1ull << m);
        }
        const std::string P_ = g.P(i), L_ = g.L(i);
        o << "; e += w * (double)(" << P_ << ".x * " << P_ << ".x + " << P_ << ".y * " << P_ << ".y); " << L_
          << ".x = (R)w * " << P_ << ".x; " << L_ << ".y = (R)w * " << P_ << ".y; }\n";
      }
      o << "}\n";
      regs_live = true;
    } else if (fused) {
      // readout + λ = wψ on the registers (tile index of logical register i =
      // deposit(i, R) | deposit(tid, S))
      const std::vector<int> S = Sbits(WL), R = Rbits(WL);
      o << "{ double wb = 0.0; for (int i = 0; i < p.n_measured; ++i) if ((base >> p.measured[i]) & 1ull) "
           "wb += (double)(1ull << i);\n";
      for (int s2 = 0; s2 < tbits; ++s2) o << "if ((tid >> " << s2 << ") & 1) wb += wt[" << S[s2] << "];\n";
      for (int i = 0; i < g.N; ++i) {
        o << "{ const double w = wb";
        for (int r = 0; r < g.RB; ++r)
          if (i >> r & 1) o << " + wt[" << R[r] << "]";
        const std::string P_ = g.P(i), L_ = g.L(i);
        o << "; e += w * (double)(" << P_ << ".x * " << P_ << ".x + " << P_ << ".y * " << P_ << ".y); " << L_
          << ".x = (R)w * " << P_ << ".x; " << L_ << ".y = (R)w * " << P_ << ".y; }\n";
      }
      o << "}\n";
      regs_live = true;  // continue into the backward windows (block stays open)
    } else if (last) {
      o << "{ double wb = 0.0; for (int i = 0; i < p.n_measured; ++i) if ((base >> p.measured[i]) & 1ull) "
           "wb += (double)(1ull << i);\n"
        << "for (int bb = 0; bb < Q - " << g.RB << "; ++bb) if ((tid >> bb) & 1) wb += wt[bb];\n";
      for (int i = 0; i < g.N; ++i) {
        o << "{ double w = wb";
        for (int b2 = 0; b2 < g.RB; ++b2)
          if (i >> b2 & 1) o << " + wt[" << (g.Q - g.RB + b2) << "]";
        o << "; const C z = tp[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u]; const uint64_t g2 = base | ot | "
          << hex64(hi_off(i)) << ";";
        if (pl->perm) {
          // folded trailing permutation: weight of P(g2), amplitude lands at P(g2)
          o << " w = 0.0";
          for (size_t m = 0; m < pl->host_measured.size(); ++m) {
            const int q = pl->host_measured[m];
            o << " + (double)((__popcll(g2 & " << hex64(pl->perm_mask[q]) << ") + " << pl->perm_const[q]
              << ") & 1) * " << (double)(1ull << m);
          }
          o << ";";
        }
        o << " e += w * (double)(z.x * z.x + z.y * z.y); gout[g2] = z;"
          << " if (glam) { C y; y.x = (R)w * z.x; y.y = (R)w * z.y; glam[g2] = y; }"
          << " if (a.state) { double* dst = a.state + v * ((int64_t)1 << p.n_qubits) * 2; uint64_t gs = g2;";
        if (pl->perm)
          o << " gs = 0; for (int q_ = 0; q_ < p.n_qubits; ++q_) gs |= (uint64_t)((__popcll(g2 & p.perm_mask[q_]) + "
               "p.perm_const[q_]) & 1) << q_;";
        o << " dst[2 * gs] = (double)z.x * gph[0] - (double)z.y * gph[1]; "
             "dst[2 * gs + 1] = (double)z.x * gph[1] + (double)z.y * gph[0]; } }\n";
      }
      o << "}\n";
    } else if (!direct_ok(WL)) {
      for (int i = 0; i < g.N; ++i)
        o << "gout[base | ot | " << hex64(hi_off(i)) << "] = tp[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u];\n";
    }
  }
  if (bwd) {
    const WinHost& WL = P.hwins[nwin - 1];
    if (!fused) {
      identity_map();
      if (direct_ok(WL)) {
        o << "{ // window " << nwin - 1 << " (adjoint): direct load\n";
        g.ph_decl = false;
        g.win_tb(WL, tbits);
        direct_load(WL, true);
        regs_live = true;
      } else {
        for (int i = 0; i < g.N; ++i) o << "p" << i << " = gpsi[base | ot | " << hex64(hi_off(i)) << "];\n";
        for (int i = 0; i < g.N; ++i) o << "l" << i << " = glam[base | ot | " << hex64(hi_off(i)) << "];\n";
        for (int i = 0; i < g.N; ++i) o << "tp[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u] = p" << i << ";\n";
        for (int i = 0; i < g.N; ++i) o << "tl[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u] = l" << i << ";\n";
        gsync();
        regs_live = false;
      }
    }
    bool bwd_shfl_in = false;   // this window's registers arrive by shuffles
    for (int wi = 0; wi < nwin; ++wi) {
      const int w = nwin - 1 - wi;
      if (first && w < stop_win) break;
      const WinHost& W = P.hwins[w];
      const bool cont = wi == 0 && regs_live;  // block already open, registers hold window w
      if (!cont) {
        o << "{ // window " << w << " (adjoint)\n";
        g.ph_decl = false;
        g.win_tb(W, tbits);
        if (!bwd_shfl_in) {
          identity_map();
          if (!(ablate & 1)) {
            g.load_regs(W, "p", "tp");
            g.load_regs(W, "l", "tl");
          }
        }
      }
      bwd_shfl_in = false;
      g.pending = false;
      const int lo = std::max<int>(W.op0, first ? stop_op : 0);
      std::vector<int> ks;
      for (int k = W.op1 - 1; k >= lo; --k) ks.push_back(k);
      hoist(ks);
      if (std::getenv("HQ_JIT_OPS")) {
        std::fprintf(stderr, "bwd win %d:", w);
        // gate letter (H X Y Z, x y z = RX RY RZ, C = CNOT, c = CZ, R = CR, S = SWAP), codes, ' = derivative
        for (int k : ks) {
          const WOp& q = P.wops[k];
          std::fprintf(stderr, " %c%d", "HXYZxyzCcRS"[q.kind], q.a);
          if (q.b >= 0) std::fprintf(stderr, ",%d", q.b);
          if (q.dl >= 0) std::fprintf(stderr, "'");
        }
        std::fprintf(stderr, "\n");
      }
      const bool end = first ? (wi == nwin - 1 || w == stop_win) : (w == 0);
      pp_acquire();
      if (end) {
        emit_steps(ks, 0, true, [&] {
          g.flush_batch();
          g.flush_vph(true);
          g.flush_pending(true);
          pp_release(true);
          if (fold_end) {
            // λ at the circuit start (all first-pass gates un-applied), contracted
            // with the tile's initial factors z_q (fz):
            //   lamN[t] = Σ_i λ[t, i] conj(Π_b z_{local[b]}[bit_b(i)])      (non-tile folded qubits)
            //   A_q[c](t) = Σ_{i: bit_q(i)=c} λ[t, i] conj(Π_{b≠q} z[..])   (tile folded qubits q)
            // per register window: i = (register index r, thread index) with
            // W_R(r) = Π over register qubits, wt_ = Π over thread qubits
            const std::vector<int> S = Sbits(W), Rr = Rbits(W);
            const int nlq = (int)pl->fold_local.size();
            const int NV = 2 + 4 * nlq;   // doubles reduced per tile
            auto fzr = [&](int tilebit, const std::string& bit) {
              return "fz[" + std::to_string(2 * P.local[tilebit]) + " + (" + bit + ")]";
            };
            auto wreg = [&](int i, int skip) {   // product of register factors of index i, skipping register bit skip
              std::string e = "one_";
              for (int r = 0; r < g.RB; ++r)
                if (r != skip) e = "cm_(" + e + ", " + fzr(Rr[r], std::to_string((i >> r) & 1)) + ")";
              return e;
            };
            auto cjacc = [&](const std::string& acc, const std::string& w, const std::string& l) {
              return acc + ".x += " + w + ".x * " + l + ".x + " + w + ".y * " + l + ".y; " + acc + ".y += " + w +
                     ".x * " + l + ".y - " + w + ".y * " + l + ".x;";
            };
            o << "{ C one_; one_.x = (R)1; one_.y = (R)0;\nC wt_ = one_;\n";
            for (int s2 = 0; s2 < tbits; ++s2)
              o << "wt_ = cm_(wt_, " << fzr(S[s2], "(tid >> " + std::to_string(s2) + ") & 1") << ");\n";
            o << "C T_; T_.x = (R)0; T_.y = (R)0;\n";
            for (int i = 0; i < g.N; ++i) o << "{ const C w_ = " << wreg(i, -1) << "; " << cjacc("T_", "w_", g.L(i)) << " }\n";
            o << "double vv_[" << NV << "];\n"
              << "vv_[0] = (double)(wt_.x * T_.x + wt_.y * T_.y); vv_[1] = (double)(wt_.x * T_.y - wt_.y * T_.x);\n";
            for (int k2 = 0; k2 < nlq; ++k2) {
              const int q = pl->fold_local[k2];
              int tb = -1;
              for (int b2 = 0; b2 < g.Q; ++b2)
                if (P.local[b2] == q) tb = b2;
              int rpos = -1, spos = -1;
              for (int r = 0; r < g.RB; ++r)
                if (Rr[r] == tb) rpos = r;
              for (int s2 = 0; s2 < tbits; ++s2)
                if (S[s2] == tb) spos = s2;
              const int v0 = 2 + 4 * k2;
              if (rpos >= 0) {
                for (int c = 0; c < 2; ++c) {
                  o << "{ C a_; a_.x = (R)0; a_.y = (R)0;\n";
                  for (int i = 0; i < g.N; ++i)
                    if (((i >> rpos) & 1) == c)
                      o << "{ const C w_ = " << wreg(i, rpos) << "; " << cjacc("a_", "w_", g.L(i)) << " }\n";
                  o << "vv_[" << v0 + 2 * c << "] = (double)(wt_.x * a_.x + wt_.y * a_.y); vv_[" << v0 + 2 * c + 1
                    << "] = (double)(wt_.x * a_.y - wt_.y * a_.x); }\n";
                }
              } else {
                o << "{ C e_ = one_;";
                for (int s2 = 0; s2 < tbits; ++s2)
                  if (s2 != spos) o << " e_ = cm_(e_, " << fzr(S[s2], "(tid >> " + std::to_string(s2) + ") & 1") << ");";
                o << "\nconst double xr_ = (double)(e_.x * T_.x + e_.y * T_.y), xi_ = (double)(e_.x * T_.y - e_.y * T_.x);\n"
                  << "const bool b_ = (tid >> " << spos << ") & 1;\n"
                  << "vv_[" << v0 << "] = b_ ? 0.0 : xr_; vv_[" << v0 + 1 << "] = b_ ? 0.0 : xi_; vv_[" << v0 + 2
                  << "] = b_ ? xr_ : 0.0; vv_[" << v0 + 3 << "] = b_ ? xi_ : 0.0; }\n";
              }
            }
            o << "#pragma unroll\nfor (int k_ = 0; k_ < " << NV << "; ++k_) vv_[k_] = warp_sum<double>(vv_[k_]);\n";
            sync();
            o << "if ((tid & 31) == 0) { for (int k_ = 0; k_ < " << NV << "; ++k_) fred[(tidw >> 5) * " << NV
              << " + k_] = vv_[k_]; }\n";
            sync();
            o << "if (tid < " << NV / 2 << ") { double ax = 0.0, ay = 0.0; for (int k = 0; k < " << nw
              << "; ++k) { ax += fred[(grp * " << nw << " + k) * " << NV << " + 2 * tid]; ay += fred[(grp * " << nw
              << " + k) * " << NV << " + 2 * tid + 1]; }\n"
              << "if (tid == 0) { double* dst = a.lamN + 2 * (vl * ((int64_t)1 << " << nonlocal.size()
              << ") + (int64_t)t); dst[0] = ax; dst[1] = ay; }\n";
            if (nlq) {
              // weight the tile by conj(Π over its tile-id qubits of z) and keep per CTA
              o << "else { double fx = 1.0, fy = 0.0;";
              for (size_t i2 = 0; i2 < nonlocal.size(); ++i2)
                o << " { const C z_ = fz[" << 2 * nonlocal[i2] << " + ((t >> " << i2
                  << ") & 1)]; const double nx = fx * (double)z_.x - fy * (double)z_.y; fy = fx * (double)z_.y + fy * (double)z_.x; fx = nx; }";
              o << "\nlacc_x += fx * ax + fy * ay; lacc_y += fx * ay - fy * ax; } }\n";
            } else {
              o << "}\n";
            }
            sync();
            o << "}\n";
          }
          if (first) return;
          if (direct_ok(W)) {
            direct_store(W, true);
          } else {
            pre_store_sync();
            g.store_regs(W, "p", "tp");
            g.store_regs(W, "l", "tl");
            sync();
            for (int i = 0; i < g.N; ++i) {
              o << "if (gout) gout[base | ot | " << hex64(hi_off(i)) << "] = tp[tpad + " << Gen::pad((uint32_t)(i * g.T))
                << "u];\n";
              o << "glam[base | ot | " << hex64(hi_off(i)) << "] = tl[tpad + " << Gen::pad((uint32_t)(i * g.T)) << "u];\n";
            }
          }
        }, ubudget);
        o << "}\n";
        break;
      }
      std::vector<std::pair<int, int>> sw;
      std::vector<int> perm;
      const bool to_shfl = w > 0 && shfl_ok(W, P.hwins[w - 1], sw, perm);
      emit_steps(ks, 0, true, [&] {
        g.flush_batch();
        g.flush_vph(true);
        g.flush_pending(true);
        pp_release(false);
        if (ablate & 1) return;
        if (to_shfl) {
          emit_shfl(sw, perm, true);
          return;
        }
        pre_store_sync();
        g.store_regs(W, "p", "tp");
        g.store_regs(W, "l", "tl");
        post_store_sync(W, P.hwins[w - 1]);
      }, ubudget);
      o << "}\n";
      if (to_shfl) identity_map();   // every branch path ended canonical
      bwd_shfl_in = to_shfl;
    }
  }
  gsync();
  o << "}\n";  // tile loop
  if (fwd && last)
    o << "e = block_sum<R>(e, red, tid, T);\nif (tid == 0) ps.rpart[vl * ps.n_chunks + chunk] = e;\n";
  if (fold_end && !pl->fold_local.empty())
    o << "if (tid >= 1 && tid < " << 1 + 2 * pl->fold_local.size() << ") { double* dst = a.locpart + 2 * ((vl * ps.n_chunks + "
         "chunk) * " << 2 * pl->fold_local.size() << " + (tid - 1)); dst[0] = lacc_x; dst[1] = lacc_y; }\n";
  if (bwd && pp && L.per_thread) {
    // ping-pong, per-thread mode: every partial is in registers (reg_acc ==
    // n_dslots): per-warp sums, then one warp per slot folds the CTA's warps
    for (int k = 0; k < reg_acc; ++k)
      o << "{ const double s_ = warp_sum<double>((double)da" << k << "); if ((tid & 31) == 0) dacc[" << k << " * "
        << nwt << " + (tidw >> 5)] = (R)s_; }\n";
    o << "__syncthreads();\n{ const int lane_ = tid & 31;\nfor (int i = tidw >> 5; i < " << P.n_dslots_pass
      << "; i += " << nwt << ") { double s = 0.0; for (int k = lane_; k < " << nwt
      << "; k += 32) s += (double)dacc[i * " << nwt << " + k]; s = warp_sum<double>(s); "
      << "if (lane_ == 0) a.dpart[((int64_t)v * p.n_adj + ps.dlist[i]) * a.n_parts + chunk] = s; } }\n";
  } else if (bwd) {
    const int width = nwt * L.group;
    for (int k = 0; k < reg_acc; ++k) o << "dacc[" << k << " * T + tid] = da" << k << ";\n";
    // one warp per slot: lanes sum strided partials in double, then a shuffle tree
    o << "__syncthreads();\n{ const int lane_ = tid & 31;\nfor (int i = tidw >> 5; i < " << P.n_dslots_pass
      << "; i += " << nwt << ") { double s = 0.0; for (int k = lane_; k < " << width
      << "; k += 32) s += (double)dacc[i * " << L.slot_stride << " + k]; s = warp_sum<double>(s); "
      << "if (lane_ == 0) a.dpart[((int64_t)v * p.n_adj + ps.dlist[i]) * a.n_parts + chunk] = s; } }\n";
  }
  o << "}\n";
  std::string body = o.str();
  std::string decl, build;
  if (!g.ptab.empty()) {
    const std::string nm = std::string(fused ? "hq_fb" : (bwd ? "hq_b" : "hq_f")) + std::to_string(pi);
    std::ostringstream d, b;
    std::vector<int> off{0}, sl, mu;
    for (const auto& m : g.ptab) {
      for (const auto& kv : m) { sl.push_back(kv.first); mu.push_back(kv.second); }
      off.push_back((int)sl.size());
    }
    auto arr = [&](const char* ty, const char* tag, const std::vector<int>& v) {
      d << "__device__ const " << ty << " " << nm << tag << "[" << v.size() << "] = {";
      for (size_t i = 0; i < v.size(); ++i) d << (i ? "," : "") << v[i];
      d << "};\n";
    };
    arr("short", "_pto", off);
    arr("short", "_pts", sl);
    arr("signed char", "_ptk", mu);
    decl = d.str();
    const int K = (int)g.ptab.size();
    b << "__shared__ C ptab_[" << K << "];\n" << (g.shear_ph ? "__shared__ int ptsg_[" + std::to_string(K) + "];\n" : "")
      << "for (int j_ = tidw; j_ < " << K << "; j_ += " << L.block << ") { R x_ = (R)1, y_ = (R)0;\n"
      << "  for (int m_ = " << nm << "_pto[j_]; m_ < " << nm << "_pto[j_ + 1]; ++m_) { const int s_ = " << nm
      << "_pts[m_], k_ = " << nm << "_ptk[m_];\n"
      << "    if (s_ < 0) { x_ = -x_; y_ = -y_; continue; }\n"
      << "    const R c_ = trig[8 * s_ + 2], sn_ = k_ < 0 ? -trig[8 * s_ + 3] : trig[8 * s_ + 3];\n"
      << "    for (int r_ = 0; r_ < (k_ < 0 ? -k_ : k_); ++r_) { const R t_ = x_ * c_ - y_ * sn_; y_ = x_ * sn_ + y_ * c_; "
         "x_ = t_; } }\n"
      << (g.shear_ph
              ? "  { double f_ = atan2((double)y_, (double)x_); int ng_ = 0;\n"
                "    if (f_ > 1.5707963267948966) { f_ -= 3.141592653589793; ng_ = (int)0x80000000; }\n"
                "    else if (f_ < -1.5707963267948966) { f_ += 3.141592653589793; ng_ = (int)0x80000000; }\n"
                "    ptab_[j_].x = (R)(-tan(0.5 * f_)); ptab_[j_].y = (R)sin(f_); ptsg_[j_] = ng_; } }\n__syncthreads();\n"
              : "  ptab_[j_].x = x_; ptab_[j_].y = y_; }\n__syncthreads();\n");
    build = b.str();
  }
  body.replace(body.find("/*HQ_PTAB_BUILD*/"), std::strlen("/*HQ_PTAB_BUILD*/"), build);
  return decl + body;
}

// One thread per (virtual) sample for the smallest circuits (n ≤ 4): the
// whole state and λ in registers (2^n each), every gate a compile-time
// register operation (renamings, shears, phases), derivative dots into
// register accumulators.  Readout / gradients only; initial states, state
// loads and amplitude output stay with the interpreter.
static std::string gen_small(const hq_plan_s* pl) {
  const bool c64 = pl->precision == HQ_C64;
  Gen g;
  g.RB = pl->n_qubits;
  g.N = 1 << g.RB;
  g.Q = pl->n_qubits;
  g.T = 1;
  g.c64 = c64;
  g.packed = c64 && !std::getenv("HQ_NO_F32X2");
  g.exact = false;
  g.map.assign(g.N, 0);
  for (int i = 0; i < g.N; ++i) g.map[i] = i;
  std::ostringstream& o = g.o;
  const int A = std::max(1, pl->n_slots);
  std::vector<WOp> wops;
  std::vector<int> dslot_of_dl;
  for (const DOp& d : pl->dops) {
    WOp w{};
    w.kind = (int8_t)d.kind;
    w.a = (int8_t)d.a;
    w.b = (int8_t)d.b;
    w.slot = (int16_t)d.slot;
    w.dl = -1;
    if (d.dslot >= 0) {
      w.dl = (int16_t)dslot_of_dl.size();
      dslot_of_dl.push_back(d.dslot);
    }
    wops.push_back(w);
  }
  const int K = (int)dslot_of_dl.size();
  o << "extern \"C\" __global__ void __launch_bounds__(128) hq_small(const hq::KArgs a) {\n"
    << "using namespace hq;\n"
    << "typedef " << g.R() << " R; typedef " << (c64 ? "float2" : "double2") << " C;\n"
    << "const R HH = (R)0.70710678118654752440;\n(void)HH;\n"
    << "const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;\nif (v >= a.V) return;\n"
    << "const DevPlan& p = a.p;\nconst VSample vs = decode_vsample(p, v, a.B);\n"
    << "const double* xr = a.x + vs.b * a.ldx;\n"
    << "R trig[" << 8 * A << "];\n"
    << "for (int i = 0; i < p.n_slots; ++i) { const double sv = eval_slot(p, i, xr, a.theta, vs.shvar, vs.shval); "
       "double sn, cs; sincos(0.5 * sv, &sn, &cs); const double sg = cs < 0.0 ? -1.0 : 1.0; "
       "const double c2 = sg * cs, s2 = sg * sn; trig[8 * i] = (R)cs; trig[8 * i + 1] = (R)sn; "
       "trig[8 * i + 2] = (R)(cs * cs - sn * sn); trig[8 * i + 3] = (R)(2.0 * cs * sn); "
       "trig[8 * i + 4] = (R)(-s2 / (1.0 + c2)); trig[8 * i + 5] = (R)s2; trig[8 * i + 6] = (R)sg; "
       "trig[8 * i + 7] = (R)0; }\n";
  o << "C";
  for (int i = 0; i < g.N; ++i) o << (i ? ", " : " ") << "p" << i;
  o << ";\n";
  for (int i = 0; i < g.N; ++i) o << "p" << i << ".x = (R)" << (i == 0 ? 1 : 0) << "; p" << i << ".y = (R)0;\n";
  for (const WOp& w : wops) g.apply(w, false, false);
  g.flush_pending(false);
  // readout weights: w(i) = Σ_k 2^k bit(i, measured[k])
  auto weight = [&](int i) {
    double wv = 0.0;
    for (size_t k = 0; k < pl->host_measured.size(); ++k)
      if ((i >> pl->host_measured[k]) & 1) wv += (double)(1ull << k);
    return wv;
  };
  o << "double e = 0.0;\n";
  for (int i = 0; i < g.N; ++i) {
    const double wv = weight(i);
    if (wv != 0.0)
      o << "e += " << wv << " * (double)(" << g.P(i) << ".x * " << g.P(i) << ".x + " << g.P(i) << ".y * " << g.P(i)
        << ".y);\n";
  }
  o << "if (vs.u < 0) a.out[v] = e; else a.tp[vs.u] = e;\n";
  if (K > 0) {
    o << "if (a.want_adj && vs.u < 0) {\nC";
    for (int i = 0; i < g.N; ++i) o << (i ? ", " : " ") << "l" << i;
    o << ";\n";
    for (int i = 0; i < g.N; ++i)
      o << g.L(i) << ".x = (R)" << weight(i) << " * " << g.P(i) << ".x; " << g.L(i) << ".y = (R)" << weight(i) << " * "
        << g.P(i) << ".y;\n";
    for (int k = 0; k < K; ++k) o << "R da" << k << " = (R)0;\n";
    g.pending = false;
    g.ph_decl = false;
    for (int k = (int)wops.size() - 1; k >= 0; --k) {
      g.dot(wops[k], true, 32, 1, K);
      g.apply(wops[k], true, true);
    }
    g.flush_pending(true);
    for (int k = 0; k < K; ++k)
      o << "{ double* dst = a.dpart + (v * p.n_adj + " << dslot_of_dl[k] << ") * a.n_parts; dst[0] = (double)da" << k
        << "; for (int q_ = 1; q_ < a.n_parts; ++q_) dst[q_] = 0.0; }\n";
    o << "}\n";
  }
  o << "}\n";
  return o.str();
}

namespace {

struct Unit {
  std::string src;
  uint64_t hash = 0;
  std::vector<char> cubin;
  std::string err;
  bool need_compile = false;
};

void compile_unit(Nvrtc& nv, Unit& u) {
  nvrtcProgram prog = nullptr;
  if (nv.create(&prog, u.src.c_str(), "hq_jit.cu", 0, nullptr, nullptr) != 0) {
    u.err = "nvrtcCreateProgram failed";
    return;
  }
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true"};
  const int rc = nv.compile(prog, 4, opts);
  if (rc != 0) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    u.err = "nvrtc compile failed: " + log.substr(0, 4000);
  } else {
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    u.cubin.resize(cs);
    nv.cubin(prog, u.cubin.data());
  }
  nv.destroy(&prog);
}

}  // namespace

// Build (or fetch) one cubin per pass (fwd + bwd kernels); missing cubins are
// compiled concurrently on the host cores.
hq_status jit_build(hq_plan_s* pl, std::string& err) {
  const char* env = std::getenv("HQ_JIT");
  if (env && env[0] == '0') { err = "disabled by HQ_JIT=0"; return HQ_E_CONFIG; }
  Nvrtc& nv = nvrtc();
  const bool small = pl->onchip;
  const int np = small ? 1 : (int)pl->passes.size();
  const std::string head = std::string(kHeader) + kJitPod + kJitDev + kHelpers;
  std::vector<Unit> units(np);
  std::string dump;
  for (int i = 0; i < np; ++i) {
    const bool fused_i = i == np - 1 && !pl->seg;
    units[i].src = small ? head + gen_small(pl)
                         : head + gen_pass(pl, i, 0) + gen_pass(pl, i, 1) + (fused_i ? gen_pass(pl, i, 2) : "");
    // keyed by source AND compiler version (different NVRTCs -> different code)
    units[i].hash = fnv1a(units[i].src + "\n// nvrtc " + std::to_string(nv.major) + "." + std::to_string(nv.minor));
    if (std::getenv("HQ_JIT_DUMP")) dump += units[i].src;
  }
  if (const char* path = std::getenv("HQ_JIT_DUMP")) {
    std::ofstream f(path);
    f << dump;
  }
  const std::string dir = cache_dir();
  auto path_of = [&](uint64_t h) {
    char name[64];
    std::snprintf(name, sizeof name, "/%016llx.sm_100a.cubin", (unsigned long long)h);
    return dir + name;
  };
  std::vector<int> todo;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int i = 0; i < np; ++i) {
      if (g_libs.count(units[i].hash)) continue;
      if (!read_file(path_of(units[i].hash), units[i].cubin)) { units[i].need_compile = true; todo.push_back(i); }
    }
  }
  if (!todo.empty()) {
    if (!nv.ok) { err = nv.why; return HQ_E_CONFIG; }
    unsigned nthr = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("HQ_JIT_THREADS")) nthr = (unsigned)std::atoi(e);
    if (nthr < 1) nthr = 1;
    nthr = std::min<unsigned>(nthr, (unsigned)todo.size());
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthr; ++t)
      pool.emplace_back([&]() {
        for (size_t k; (k = next.fetch_add(1)) < todo.size();) compile_unit(nv, units[todo[k]]);
      });
    for (auto& th : pool) th.join();
    for (int i : todo) {
      if (!units[i].err.empty()) { err = units[i].err; return HQ_E_CUDA; }
      write_file(path_of(units[i].hash), units[i].cubin);
    }
  }
  if (std::getenv("HQ_JIT_COMPILE_ONLY")) { err = "compile-only"; return HQ_E_CONFIG; }
  if (small) {
    cudaLibrary_t lib = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_libs.find(units[0].hash);
      if (it != g_libs.end()) lib = it->second;
    }
    if (!lib) {
      cudaError_t ce = cudaLibraryLoadData(&lib, units[0].cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
      if (ce != cudaSuccess) {
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
        return HQ_E_CUDA;
      }
      std::lock_guard<std::mutex> lk(g_mu);
      g_libs[units[0].hash] = lib;
    }
    if (cudaLibraryGetKernel(&pl->jit.small, lib, "hq_small") != cudaSuccess) {
      err = "generated kernel missing";
      return HQ_E_CUDA;
    }
    return HQ_OK;
  }
  pl->jit.fwd.assign(np, nullptr);
  pl->jit.bwd.assign(np, nullptr);
  for (int m = 0; m < 3; ++m) {
    pl->jit.block[m].assign(np, 0);
    pl->jit.smem[m].assign(np, 0);
  }
  for (int i = 0; i < np; ++i) {
    cudaLibrary_t lib = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_libs.find(units[i].hash);
      if (it != g_libs.end()) lib = it->second;
    }
    if (!lib) {
      cudaError_t ce = cudaLibraryLoadData(&lib, units[i].cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
      if (ce != cudaSuccess) {
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
        return HQ_E_CUDA;
      }
      std::lock_guard<std::mutex> lk(g_mu);
      g_libs[units[i].hash] = lib;
    }
    const std::string s = std::to_string(i);
    if (cudaLibraryGetKernel(&pl->jit.fwd[i], lib, ("hq_f" + s).c_str()) != cudaSuccess ||
        cudaLibraryGetKernel(&pl->jit.bwd[i], lib, ("hq_b" + s).c_str()) != cudaSuccess ||
        (i == np - 1 && !pl->seg && cudaLibraryGetKernel(&pl->jit.fused, lib, ("hq_fb" + s).c_str()) != cudaSuccess)) {
      err = "generated kernel missing";
      return HQ_E_CUDA;
    }
    for (int mode = 0; mode < (i == np - 1 && !pl->seg ? 3 : 2); ++mode) {
      const JitLayout L = jit_layout(pl, i, mode != 0, mode == 2);
      pl->jit.block[mode][i] = L.block;
      pl->jit.smem[mode][i] = L.total;
      cudaKernel_t k = mode == 0 ? pl->jit.fwd[i] : (mode == 1 ? pl->jit.bwd[i] : pl->jit.fused);
      cudaError_t ce = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
      if (ce != cudaSuccess) {
        err = std::string("smem attribute: ") + cudaGetErrorString(ce);
        return HQ_E_CUDA;
      }
    }
  }
  pl->jit.ok = true;
  return HQ_OK;
}

cudaError_t jit_launch_small(const hq_plan_s* pl, const KArgs& a, cudaStream_t st) {
  KArgs ac = a;
  void* args[] = {&ac};
  return cudaLaunchKernel((const void*)pl->jit.small, dim3((unsigned)((a.V + 127) / 128)), dim3(128), args, 0, st);
}

cudaError_t jit_launch_pass(const hq_plan_s* pl, int i, int mode, const KArgs& a, const JPass& ps,
                            unsigned grid, cudaStream_t st) {
  const bool bwd = mode != 0;
  cudaKernel_t k = mode == 0 ? pl->jit.fwd[i] : (mode == 1 ? pl->jit.bwd[i] : pl->jit.fused);
  const int T = pl->jit.block[mode][i];
  const size_t smem = pl->jit.smem[mode][i];
  KArgs ac = a;
  JPass pc = ps;
  void* args[] = {&ac, &pc};
  cudaError_t e = cudaLaunchKernel((const void*)k, dim3(grid), dim3(T), args, smem, st);
  if (e != cudaSuccess && std::getenv("HQ_JIT_DEBUG")) {
    cudaFuncAttributes fa{};
    cudaError_t e2 = cudaFuncGetAttributes(&fa, (const void*)k);
    std::fprintf(stderr, "hq_jit launch %s%d grid=%u block=%d smem=%zu -> %s | attrs(%s): regs=%d maxthr=%d "
                 "static_smem=%zu maxdyn=%d local=%zu\n", bwd ? "hq_b" : "hq_f", i, grid, T, smem,
                 cudaGetErrorString(e), cudaGetErrorString(e2), fa.numRegs, fa.maxThreadsPerBlock,
                 fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.localSizeBytes);
  }
  return e;
}

}  // namespace hq
