// jit_program.cu -- fused element-wise EXPRESSION PROGRAMS (Schur %, /,
// abs, scalar +, nested linear combinations) compiled to one streaming
// kernel per program shape at run time.
//
// This is the B200 counterpart of Armadillo's expression templates: the
// planner (paper_2502_03000_b200/elementwise.py) lowers a connected
// element-wise region to a postfix program; here the program becomes
// straight-line CUDA source, NVRTC compiles it for sm_100a once per
// (dtype, program, layout) and the cubin is cached for the process.
// Constants are kernel arguments, so 2*A + B%C and 3*A + B%C share one
// kernel.  Semantics per element = naive_evaluate (expr.py:304-391) with
// the reference's R1 coefficient folding (rewrite.py:265-298): one IEEE
// rounding per node, explicit __d*_rn intrinsics, no FMA.
//
// Traffic: (nsrc + 1) * n_elems * sizeof(T) -- every source once, the
// result once, no temporaries; 16-byte vector loads, 2 vectors per
// source in flight per thread.
#include <nvrtc.h>

#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace lm {

namespace {

enum Op { OP_LOAD = 0, OP_CONST = 1, OP_ADD = 2, OP_SUB = 3, OP_MUL = 4, OP_DIV = 5, OP_ABS = 6, OP_NEG = 7 };

struct JitEntry {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
};

std::mutex g_mu;
std::unordered_map<std::string, JitEntry> g_cache;

// Straight-line body of  T f(T x0..x{nsrc-1}) ; constants k{i} are
// kernel parameters captured by the lambda-free macro expansion below.
int gen_body(int nins, const int32_t *ops, const int32_t *args, int nsrc, int nconst, std::string &body) {
    std::vector<std::string> st;
    std::ostringstream os;
    int tmp = 0;
    for (int q = 0; q < nins; ++q) {
        const int op = ops[q], a = args[q];
        switch (op) {
        case OP_LOAD:
            if (a < 0 || a >= nsrc) return -1;
            st.push_back("x" + std::to_string(a));
            break;
        case OP_CONST:
            if (a < 0 || a >= nconst) return -1;
            st.push_back("((T)k" + std::to_string(a) + ")");
            break;
        case OP_ADD:
        case OP_SUB:
        case OP_MUL:
        case OP_DIV: {
            if (st.size() < 2) return -2;
            std::string rhs = st.back();
            st.pop_back();
            std::string lhs = st.back();
            st.pop_back();
            const char *fn = op == OP_ADD ? "RADD" : op == OP_SUB ? "RSUB" : op == OP_MUL ? "RMUL" : "RDIV";
            std::string t = "t" + std::to_string(tmp++);
            os << "  const T " << t << " = " << fn << "(" << lhs << ", " << rhs << ");\n";
            st.push_back(t);
            break;
        }
        case OP_ABS:
        case OP_NEG: {
            if (st.empty()) return -2;
            std::string x = st.back();
            st.pop_back();
            std::string t = "t" + std::to_string(tmp++);
            os << "  const T " << t << " = " << (op == OP_ABS ? "RABS(" : "(-") << x << ");\n";
            st.push_back(t);
            break;
        }
        default:
            return -1;
        }
    }
    if (st.size() != 1) return -3;
    os << "  return " << st.back() << ";\n";
    body = os.str();
    return 0;
}

std::string gen_source(bool f64, bool flat, int nsrc, int nconst, const std::string &body) {
    std::ostringstream s;
    s << "typedef long long i64;\n";
    if (f64) {
        s << "typedef double T;\n"
             "struct __align__(16) V { double x, y; };\n"
             "#define VN 2\n"
             "#define RADD __dadd_rn\n#define RSUB __dsub_rn\n#define RMUL __dmul_rn\n#define RDIV __ddiv_rn\n"
             "__device__ __forceinline__ T RABS(T v) { return __longlong_as_double(__double_as_longlong(v) & "
             "0x7fffffffffffffffLL); }\n"
             "__device__ __forceinline__ V ldv(const T* p) { V r; asm volatile(\"ld.global.nc.L1::no_allocate.v2.f64 "
             "{%0, %1}, [%2];\" : \"=d\"(r.x), \"=d\"(r.y) : \"l\"(p)); return r; }\n"
             "__device__ __forceinline__ void stv(T* p, V v) { asm volatile(\"st.global.cs.v2.f64 [%0], {%1, %2};\" "
             ":: \"l\"(p), \"d\"(v.x), \"d\"(v.y) : \"memory\"); }\n";
    } else {
        s << "typedef float T;\n"
             "struct __align__(16) V { float x, y, z, w; };\n"
             "#define VN 4\n"
             "#define RADD __fadd_rn\n#define RSUB __fsub_rn\n#define RMUL __fmul_rn\n#define RDIV __fdiv_rn\n"
             "__device__ __forceinline__ T RABS(T v) { return __int_as_float(__float_as_int(v) & 0x7fffffff); }\n"
             "__device__ __forceinline__ V ldv(const T* p) { V r; asm volatile(\"ld.global.nc.L1::no_allocate.v4.f32 "
             "{%0, %1, %2, %3}, [%4];\" : \"=f\"(r.x), \"=f\"(r.y), \"=f\"(r.z), \"=f\"(r.w) : \"l\"(p)); return r; }\n"
             "__device__ __forceinline__ void stv(T* p, V v) { asm volatile(\"st.global.cs.v4.f32 [%0], {%1, %2, %3, "
             "%4};\" :: \"l\"(p), \"f\"(v.x), \"f\"(v.y), \"f\"(v.z), \"f\"(v.w) : \"memory\"); }\n";
    }
    // the element function
    s << "__device__ __forceinline__ T f(";
    for (int k = 0; k < nsrc; ++k) s << "T x" << k << ", ";
    for (int k = 0; k < nconst; ++k) s << "double k" << k << ", ";
    s << "int _dummy) {\n" << body << "}\n";
    auto emit_call = [&](const char *lane_fmt) {
        std::ostringstream c;
        c << "f(";
        for (int k = 0; k < nsrc; ++k) {
            char buf[128];
            snprintf(buf, sizeof(buf), lane_fmt, k, k, k);
            c << buf << ", ";
        }
        for (int k = 0; k < nconst; ++k) c << "k" << k << ", ";
        c << "0)";
        return c.str();
    };
    s << "extern \"C\" __global__ void __launch_bounds__(256) lm_prog(";
    for (int k = 0; k < nsrc; ++k) s << "const T* __restrict__ s" << k << ", ";
    s << "T* __restrict__ out, i64 rows, i64 n";
    if (!flat) {
        for (int k = 0; k < nsrc; ++k) s << ", i64 rs" << k << ", i64 cs" << k;
        s << ", i64 ors, i64 ocs";
    }
    for (int k = 0; k < nconst; ++k) s << ", double k" << k;
    s << ") {\n"
         "  const i64 nth = (i64)gridDim.x * blockDim.x;\n"
         "  i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;\n";
    if (flat) {
        s << "  const i64 nvec = n / VN;\n"
             "  for (; v + nth < nvec; v += 2 * nth) {\n";
        for (int k = 0; k < nsrc; ++k)
            s << "    const V a" << k << " = ldv(s" << k << " + v * VN), b" << k << " = ldv(s" << k
              << " + (v + nth) * VN);\n";
        s << "    V ra, rb;\n"
             "    #pragma unroll\n"
             "    for (int e = 0; e < VN; ++e) {\n"
             "      (&ra.x)[e] = "
          << emit_call("(&a%d.x)[e]") << ";\n"
          << "      (&rb.x)[e] = " << emit_call("(&b%d.x)[e]") << ";\n"
          << "    }\n"
             "    stv(out + v * VN, ra); stv(out + (v + nth) * VN, rb);\n"
             "  }\n"
             "  for (; v < nvec; v += nth) {\n";
        for (int k = 0; k < nsrc; ++k) s << "    const V a" << k << " = ldv(s" << k << " + v * VN);\n";
        s << "    V ra;\n"
             "    #pragma unroll\n"
             "    for (int e = 0; e < VN; ++e) (&ra.x)[e] = "
          << emit_call("(&a%d.x)[e]") << ";\n"
          << "    stv(out + v * VN, ra);\n"
             "  }\n"
             "  if (blockIdx.x == 0)\n"
             "    for (i64 e = nvec * VN + threadIdx.x; e < n; e += blockDim.x) out[e] = "
          << emit_call("s%d[e]") << ";\n";
    } else {
        s << "  for (i64 e = v; e < n; e += nth) {\n"
             "    const i64 j = e / rows, i = e - j * rows;\n"
             "    out[i * ors + j * ocs] = "
          << emit_call("s%d[i * rs%d + j * cs%d]") << ";\n"
          << "  }\n";
    }
    s << "}\n";
    return s.str();
}

int compile(const std::string &src, JitEntry &out) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "lm_prog.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        set_error("nvrtcCreateProgram failed");
        return -3;
    }
    const char *opts[] = {"-arch=sm_100a", "--fmad=false", "-default-device", "-lineinfo", "--std=c++17"};
    nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        set_error("NVRTC compile failed: %s\n%s", nvrtcGetErrorString(r), log.c_str());
        nvrtcDestroyProgram(&prog);
        return -3;
    }
    size_t nbin = 0;
    nvrtcGetCUBINSize(prog, &nbin);
    std::vector<char> cubin(nbin);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    LM_CUDA(cudaLibraryLoadData(&out.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    LM_CUDA(cudaLibraryGetKernel(&out.kern, out.lib, "lm_prog"));
    return 0;
}

bool linear(const lm_view &v) {
    if (v.rows <= 1) return v.cols <= 1 || v.cs == 1;
    if (v.cols <= 1) return v.rs == 1;
    return v.rs == 1 && v.cs == v.rows;
}

}  // namespace

// Source text for a program (exposed for tests / inspection).
int program_source(int dtype, bool flat, int nins, const int32_t *ops, const int32_t *args, int nconst, int nsrc,
                   std::string &src) {
    std::string body;
    int rc = gen_body(nins, ops, args, nsrc, nconst, body);
    if (rc) {
        set_error("malformed element-wise program (%d)", rc);
        return -1;
    }
    src = gen_source(dtype == LM_F64, flat, nsrc, nconst, body);
    return 0;
}

}  // namespace lm

using namespace lm;

extern "C" int lm_fused_program(int dtype, int nins, const int32_t *ops, const int32_t *args, int nconst,
                                const double *consts, int nsrc, const lm_view *srcs, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64 || dtype == LM_F32, "bad dtype %d", dtype);
    LM_REQUIRE(nins >= 1 && nsrc >= 0 && nsrc <= 64 && nconst >= 0 && nconst <= 64, "bad program sizes");
    for (int k = 0; k < nsrc; ++k)
        LM_REQUIRE(srcs[k].rows == out.rows && srcs[k].cols == out.cols, "program source %d shape mismatch", k);
    const int64_t n = out.rows * out.cols;
    if (n == 0) return 0;
    bool flat = linear(out) && (reinterpret_cast<uintptr_t>(out.ptr) & 15) == 0;
    for (int k = 0; k < nsrc; ++k) flat = flat && linear(srcs[k]) && (reinterpret_cast<uintptr_t>(srcs[k].ptr) & 15) == 0;

    std::ostringstream key;
    key << dtype << (flat ? 'F' : 'S') << nsrc << ':' << nconst << ':';
    for (int q = 0; q < nins; ++q) key << ops[q] << ',' << args[q] << ';';
    JitEntry ent;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_cache.find(key.str());
        if (it != g_cache.end()) {
            ent = it->second;
        } else {
            std::string src;
            int rc = program_source(dtype, flat, nins, ops, args, nconst, nsrc, src);
            if (rc) return rc;
            rc = compile(src, ent);
            if (rc) return rc;
            g_cache[key.str()] = ent;
        }
    }
    // kernel arguments (order = generated signature)
    std::vector<void *> argv;
    std::vector<int64_t> ints;
    ints.reserve(8 + 2 * nsrc);
    std::vector<const void *> ptrs(nsrc + 1);
    for (int k = 0; k < nsrc; ++k) {
        ptrs[k] = srcs[k].ptr;
        argv.push_back(&ptrs[k]);
    }
    ptrs[nsrc] = out.ptr;
    argv.push_back(&ptrs[nsrc]);
    ints.push_back(out.rows);
    ints.push_back(n);
    if (!flat) {
        for (int k = 0; k < nsrc; ++k) {
            ints.push_back(srcs[k].rs);
            ints.push_back(srcs[k].cs);
        }
        ints.push_back(out.rs);
        ints.push_back(out.cs);
    }
    for (auto &v : ints) argv.push_back(&v);
    std::vector<double> kv(consts, consts + nconst);
    for (auto &v : kv) argv.push_back(&v);

    const int vn = dtype == LM_F64 ? 2 : 4;
    int64_t items = flat ? ceil_div(n / vn, 2) : n;
    int64_t blocks = ceil_div(items < 1 ? 1 : items, 256);
    const int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    LM_CUDA(cudaLaunchKernel((const void *)ent.kern, dim3((unsigned)blocks), dim3(256), argv.data(), 0,
                             as_stream(stream)));
    count_launch(1);
    return 0;
}

// Generated CUDA source of a program, for inspection (tests).
extern "C" int lm_program_source(int dtype, int flat, int nins, const int32_t *ops, const int32_t *args, int nconst,
                                 int nsrc, char *buf, int64_t buflen) {
    clear_error();
    std::string src;
    int rc = program_source(dtype, flat != 0, nins, ops, args, nconst, nsrc, src);
    if (rc) return rc;
    if ((int64_t)src.size() + 1 > buflen) return (int)src.size() + 1;
    memcpy(buf, src.c_str(), src.size() + 1);
    return 0;
}
