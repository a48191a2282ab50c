// format.cu — hybrid format signatures (Table 1 :68-82, Table 2 :297-327) and their
// expansion into tiers (see vf_internal.cuh).
#include <ctype.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "vf_internal.cuh"

namespace vf {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }
const char* last_error() { return g_err; }

namespace {

struct Parser {
  const char* s;
  size_t i = 0;
  void ws() {
    while (s[i] && isspace((unsigned char)s[i])) ++i;
  }
  bool eat(char c) {
    ws();
    if (s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  bool number(long* v) {
    ws();
    if (!isdigit((unsigned char)s[i])) return false;
    long x = 0;
    while (isdigit((unsigned char)s[i])) {
      x = x * 10 + (s[i] - '0');
      if (x > 1000000) return false;
      ++i;
    }
    *v = x;
    return true;
  }
  // cube sugar after a number: "^3" or UTF-8 superscript three (0xC2 0xB3)
  bool cube() {
    ws();
    if (s[i] == '^' && s[i + 1] == '3') {
      i += 2;
      return true;
    }
    if ((unsigned char)s[i] == 0xC2 && (unsigned char)s[i + 1] == 0xB3) {
      i += 2;
      return true;
    }
    return false;
  }
};

}  // namespace

static vf_status parse(const char* sig, vf_level* out, uint32_t cap, uint32_t* n_out) {
  if (!sig || !n_out || (!out && cap)) {
    set_error("vf_parse_format: null argument");
    return VF_ERR_INVALID_ARG;
  }
  Parser p{sig};
  uint32_t n = 0;
  for (;;) {
    p.ws();
    if (!sig[p.i]) break;
    char c = sig[p.i];
    if (!strchr("RDSGT", c) || c == 0) {
      set_error("parse error at position %zu: expected one of R D S G T, got '%c'", p.i, c);
      return VF_ERR_PARSE;
    }
    ++p.i;
    if (!p.eat('(')) {
      set_error("parse error at position %zu: expected '('", p.i);
      return VF_ERR_PARSE;
    }
    long a[4] = {0, 0, 0, 0};
    int na = 0;
    bool sugar = false;
    for (;;) {
      long v;
      if (!p.number(&v)) {
        set_error("parse error at position %zu: expected a non-negative integer", p.i);
        return VF_ERR_PARSE;
      }
      if (na >= 4) {
        set_error("parse error at position %zu: too many parameters", p.i);
        return VF_ERR_PARSE;
      }
      a[na++] = v;
      if (na == 1 && p.cube()) sugar = true;
      if (p.eat(',')) continue;
      if (p.eat(')')) break;
      set_error("parse error at position %zu: expected ',' or ')'", p.i);
      return VF_ERR_PARSE;
    }
    vf_level L;
    memset(&L, 0, sizeof(L));
    auto arity = [&](int want) -> bool {
      if (na != want) {
        set_error("parse error at position %zu: %c(...) takes %d parameter(s), got %d", p.i, c, want, na);
        return false;
      }
      return true;
    };
    switch (c) {
      case 'R':
        if (sugar) {
          if (!arity(1)) return VF_ERR_PARSE;
          a[1] = a[2] = a[0];
        } else if (!arity(3))
          return VF_ERR_PARSE;
        L.kind = VF_RAW;
        for (int k = 0; k < 3; ++k) L.log2_extent[k] = (uint8_t)(a[k] > 255 ? 255 : a[k]);
        break;
      case 'D':
        if (sugar) {
          if (!arity(2)) return VF_ERR_PARSE;
          a[3] = a[1];
          a[1] = a[2] = a[0];
        } else if (!arity(4))
          return VF_ERR_PARSE;
        L.kind = VF_DF;
        for (int k = 0; k < 3; ++k) L.log2_extent[k] = (uint8_t)(a[k] > 255 ? 255 : a[k]);
        L.df_max = (uint8_t)(a[3] > 255 ? 255 : a[3]);
        break;
      case 'S':
      case 'G':
        if (sugar || !arity(1)) {
          if (sugar) set_error("parse error at position %zu: ^3 sugar only applies to R and D", p.i);
          return VF_ERR_PARSE;
        }
        L.kind = c == 'S' ? VF_SVO : VF_SVDAG;
        L.depth = (uint8_t)(a[0] > 255 ? 255 : a[0]);
        break;
      case 'T':
        if (sugar || !arity(2)) {
          if (sugar) set_error("parse error at position %zu: ^3 sugar only applies to R and D", p.i);
          return VF_ERR_PARSE;
        }
        L.kind = VF_NTREE;
        L.log2_fanout = (uint8_t)(a[0] > 255 ? 255 : a[0]);
        L.depth = (uint8_t)(a[1] > 255 ? 255 : a[1]);
        break;
    }
    if (out && n < cap) out[n] = L;
    ++n;
  }
  if (n == 0) {
    set_error("parse error: empty signature");
    return VF_ERR_PARSE;
  }
  *n_out = n;
  if (n > cap) {
    set_error("vf_parse_format: %u levels exceed capacity %u", n, cap);
    return VF_ERR_INVALID_ARG;
  }
  return VF_OK;
}

vf_status expand_format(const vf_level* levels, uint32_t n, Format* f) {
  if (!levels || n == 0) {
    set_error("format has no levels");
    return VF_ERR_FORMAT;
  }
  if (n > VF_MAX_LEVELS) {
    set_error("format has %u levels (max %d)", n, VF_MAX_LEVELS);
    return VF_ERR_FORMAT;
  }
  *f = Format();
  f->n_levels = n;
  uint32_t nt = 0;
  for (uint32_t l = 0; l < n; ++l) {
    const vf_level& L = levels[l];
    f->levels[l] = L;
    uint32_t lf[3];
    uint32_t reps = 1;
    uint32_t kind;
    switch (L.kind) {
      case VF_RAW:
        for (int a = 0; a < 3; ++a) lf[a] = L.log2_extent[a];
        if (l > 0 && (lf[0] != lf[1] || lf[1] != lf[2])) {
          set_error("level %u R(%u,%u,%u) is not cubic: every level but the first must be cubic with "
                    "power-of-two extent (PAPER.md:267)",
                    l + 1, lf[0], lf[1], lf[2]);
          return VF_ERR_FORMAT;
        }
        for (int a = 0; a < 3; ++a)
          if (lf[a] > 12) {
            set_error("level %u: Raw extent 2^%u exceeds 4096", l + 1, lf[a]);
            return VF_ERR_FORMAT;
          }
        kind = K_RAW;
        break;
      case VF_SVO:
      case VF_SVDAG:
        if (L.depth < 1 || L.depth > 12) {
          set_error("level %u: %c(%u) depth must be in [1,12]", l + 1, L.kind == VF_SVO ? 'S' : 'G', L.depth);
          return VF_ERR_FORMAT;
        }
        lf[0] = lf[1] = lf[2] = 1;
        reps = L.depth;
        kind = L.kind == VF_SVO ? K_SVO : K_SVDAG;
        break;
      case VF_NTREE:
        if (L.log2_fanout < 1 || L.log2_fanout > 2) {
          set_error("level %u: T(%u,%u) needs log2 N in {1,2} (64-bit occupancy mask)", l + 1, L.log2_fanout, L.depth);
          return VF_ERR_FORMAT;
        }
        if (L.depth < 1) {
          set_error("level %u: T(%u,%u) depth must be >= 1", l + 1, L.log2_fanout, L.depth);
          return VF_ERR_FORMAT;
        }
        lf[0] = lf[1] = lf[2] = L.log2_fanout;
        reps = L.depth;
        kind = K_NTREE;
        break;
      case VF_DF:
        // D(W,H,D,M): a Raw grid whose cells also store the L1
        // distance to the nearest non-empty cell, capped at M; traversed as a Raw tier that
        // skips occupancy tests while the distance budget lasts
        for (int a = 0; a < 3; ++a) lf[a] = L.log2_extent[a];
        if (l > 0 && (lf[0] != lf[1] || lf[1] != lf[2])) {
          set_error("level %u D(%u,%u,%u,%u) is not cubic: every level but the first must be cubic with "
                    "power-of-two extent (PAPER.md:267)",
                    l + 1, lf[0], lf[1], lf[2], L.df_max);
          return VF_ERR_FORMAT;
        }
        for (int a = 0; a < 3; ++a)
          if (lf[a] > 12) {
            set_error("level %u: DF extent 2^%u exceeds 4096", l + 1, lf[a]);
            return VF_ERR_FORMAT;
          }
        if (L.df_max < 1) {
          set_error("level %u: D(...,M) needs M >= 1", l + 1);
          return VF_ERR_FORMAT;
        }
        kind = K_RAW;
        break;
      default:
        set_error("level %u: unknown kind %u", l + 1, L.kind);
        return VF_ERR_FORMAT;
    }
    for (uint32_t r = 0; r < reps; ++r) {
      if (nt >= VF_MAX_TIERS) {
        set_error("format expands to more than %d tiers", VF_MAX_TIERS);
        return VF_ERR_FORMAT;
      }
      Tier& T = f->tiers[nt++];
      T.kind = kind;
      for (int a = 0; a < 3; ++a) T.lf[a] = lf[a];
      T.level = l;
      T.depth = r;
      T.top = r == 0;
      T.last = r + 1 == reps;
      T.df = L.kind == VF_DF;
      T.df_max = L.kind == VF_DF ? L.df_max : 0;
      T.lc = 0;
    }
  }
  f->n_tiers = nt;
  // cell sizes bottom-up: lc(T-1) = 0, lc(t) = lc(t+1) + lf(t+1)
  f->tiers[nt - 1].lc = 0;
  for (int t = (int)nt - 2; t >= 0; --t) f->tiers[t].lc = f->tiers[t + 1].lc + f->tiers[t + 1].lf[0];
  for (int a = 0; a < 3; ++a) {
    uint32_t lg = f->tiers[0].lc + f->tiers[0].lf[a];
    if (lg > 12) {
      set_error("resolution 2^%u along axis %d exceeds 4096", lg, a);
      return VF_ERR_FORMAT;
    }
    f->dims[a] = 1u << lg;
  }
  return VF_OK;
}

TraceParams make_trace_params(const Format& f, uint32_t root) {
  TraceParams p;
  memset(&p, 0, sizeof(p));
  for (uint32_t t = 0; t < f.n_tiers; ++t) {
    const Tier& T = f.tiers[t];
    p.lc_pack |= (uint64_t)T.lc << (4 * t);
    p.lf_pack |= (uint64_t)(T.lf[0] & 15) << (4 * t);
    p.kind_pack |= T.kind << (2 * t);
    if (T.top) p.top_mask |= 1u << t;
    if (T.df) p.df_mask |= 1u << t;
    if (T.last) p.last_mask |= 1u << t;
    uint32_t top = t - T.depth;
    if (t < 8)
      p.level_top_pack_lo |= top << (4 * t);
    else
      p.level_top_pack_hi |= top << (4 * (t - 8));
  }
  // tau[h]: deepest tier tau in [1, T-1] whose node (edge 2^lc(tau-1)) contains two cells whose
  // coordinates agree above bit h, i.e. lc(tau-1) > h; 0 if none.
  for (uint32_t h = 0; h < 16; ++h) {
    uint32_t tau = 0;
    for (uint32_t t = 1; t < f.n_tiers; ++t)
      if (f.tiers[t - 1].lc > h) tau = t;
    p.tau_pack |= (uint64_t)tau << (4 * h);
  }
  for (int a = 0; a < 3; ++a) {
    p.lf0[a] = f.tiers[0].lf[a];
    p.dims[a] = (int32_t)f.dims[a];
  }
  for (uint32_t t = 0; t < f.n_tiers; ++t) {
    const Tier& T = f.tiers[t];
    const uint32_t lcn = t + 1 < f.n_tiers ? f.tiers[t + 1].lc : 0;
    const uint32_t lcp = t > 0 ? f.tiers[t - 1].lc : 15;
    const uint32_t sx = T.lf[0], sxy = T.lf[0] + T.lf[1];
    const uint32_t mb = t == 0 ? 12 : T.lf[0];
    p.tword[t] = (T.kind << TW_KIND) | (T.lc << TW_LC) | (lcn << TW_LCN) | (lcp << TW_LCP) | (sx << TW_SX) |
                 (sxy << TW_SXY) | (mb << TW_MB) | (T.last ? TW_LAST : 0u) |
                 (t + 1 == f.n_tiers ? TW_FINEST : 0u) | (T.df ? TW_DF : 0u) | (T.top ? TW_TOP : 0u);
  }
  p.n_tiers = f.n_tiers;
  p.root = root;
  p.refill = 16;  // A/B on incoherent rays (cfg4i): 16 best of 8/16/24/32
  p.chunk = 128;   // chunked trace (A/B)
  p.crefill = 16;
  return p;
}

}  // namespace vf

using namespace vf;

extern "C" {

const char* vf_last_error(void) { return vf::last_error(); }
int vf_abi_version(void) { return VF_ABI_VERSION; }

vf_status vf_parse_format(const char* sig, vf_level* out, uint32_t cap, uint32_t* n_out) {
  clear_error();
  return parse(sig, out, cap, n_out);
}

vf_status vf_format_to_string(const vf_level* levels, uint32_t n, char* buf, size_t cap) {
  clear_error();
  if (!levels || !buf || cap == 0) {
    set_error("vf_format_to_string: null argument");
    return VF_ERR_INVALID_ARG;
  }
  std::string s;
  char tmp[64];
  for (uint32_t l = 0; l < n; ++l) {
    const vf_level& L = levels[l];
    switch (L.kind) {
      case VF_RAW: snprintf(tmp, sizeof tmp, "R(%u, %u, %u)", L.log2_extent[0], L.log2_extent[1], L.log2_extent[2]); break;
      case VF_DF:
        snprintf(tmp, sizeof tmp, "D(%u, %u, %u, %u)", L.log2_extent[0], L.log2_extent[1], L.log2_extent[2], L.df_max);
        break;
      case VF_SVO: snprintf(tmp, sizeof tmp, "S(%u)", L.depth); break;
      case VF_SVDAG: snprintf(tmp, sizeof tmp, "G(%u)", L.depth); break;
      case VF_NTREE: snprintf(tmp, sizeof tmp, "T(%u, %u)", L.log2_fanout, L.depth); break;
      default: set_error("unknown level kind %u", L.kind); return VF_ERR_INVALID_ARG;
    }
    if (l) s += ' ';
    s += tmp;
  }
  if (s.size() + 1 > cap) {
    set_error("vf_format_to_string: buffer too small (%zu needed)", s.size() + 1);
    return VF_ERR_INVALID_ARG;
  }
  memcpy(buf, s.c_str(), s.size() + 1);
  return VF_OK;
}

vf_status vf_format_resolution(const vf_level* levels, uint32_t n, uint32_t dims[3]) {
  clear_error();
  Format f;
  vf_level tmp[VF_MAX_LEVELS];
  if (n > VF_MAX_LEVELS || !levels || !dims) {
    set_error("vf_format_resolution: bad arguments");
    return VF_ERR_INVALID_ARG;
  }
  for (uint32_t l = 0; l < n; ++l) {
    tmp[l] = levels[l];
  }
  vf_status st = expand_format(tmp, n, &f);
  if (st != VF_OK) return st;
  for (int a = 0; a < 3; ++a) dims[a] = f.dims[a];
  return VF_OK;
}

}  // extern "C"
