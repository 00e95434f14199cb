// Exclusive prefix sum of int32 arrays: block-local scan, scan of block totals, add-back.
// Used for cell starts (neighbors.py:127-133 does bincount + cumsum) and CSR row offsets.
#include <stdarg.h>
#include <stdlib.h>

#include "nnp_common.cuh"

static thread_local char g_last_error[512] = "";

void nnp_set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

extern "C" const char *nnp_last_error(void) { return g_last_error; }

thread_local int g_nnp_launch_count = 0;

thread_local bool t_nnp_pdl_ask = false;
int nnp_pdl_mode()
{
    static const int mode = [] {
        const char *v = getenv("NNP_PDL");
        return v ? atoi(v) : 0;
    }();
    return mode;
}
bool nnp_pdl_enabled()
{
    static const bool on = [] {
        const char *v = getenv("NNP_PDL");
        return v && v[0] == '1';      // off unless asked for: measured slower inside the step graph
    }();
    return on;
}

extern "C" int nnp_launch_count(int reset)
{
    int v = g_nnp_launch_count;
    if (reset) g_nnp_launch_count = 0;
    return v;
}

// ---- per-kernel timing with CUDA events on the launching stream
#include <map>
#include <string>
#include <vector>
namespace {
struct ProfRec {
    const char *label;
    cudaEvent_t start, stop;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof_recs;
}  // namespace

void nnp_prof_mark(const char *label, cudaStream_t stream, int begin)
{
    if (!g_prof_on) return;
    if (begin) {
        ProfRec r{label, nullptr, nullptr};
        cudaEventCreate(&r.start);
        cudaEventCreate(&r.stop);
        cudaEventRecord(r.start, stream);
        g_prof_recs.push_back(r);
    } else {
        for (size_t i = g_prof_recs.size(); i-- > 0;)
            if (g_prof_recs[i].label == label) {
                cudaEventRecord(g_prof_recs[i].stop, stream);
                break;
            }
    }
}

extern "C" int nnp_profile_begin(void)
{
    g_prof_on = true;
    return NNP_OK;
}

// Synchronises, writes "label total_ms count\n" lines into buf, clears the records.
extern "C" int nnp_profile_report(char *buf, int buf_bytes)
{
    g_prof_on = false;
    cudaDeviceSynchronize();
    std::map<std::string, std::pair<double, int>> acc;
    std::vector<std::string> order;
    for (auto &r : g_prof_recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.start, r.stop);
        if (!acc.count(r.label)) order.push_back(r.label);
        acc[r.label].first += ms;
        acc[r.label].second += 1;
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    g_prof_recs.clear();
    std::string out;
    for (auto &k : order) {
        char line[160];
        snprintf(line, sizeof(line), "%s %.6f %d\n", k.c_str(), acc[k].first, acc[k].second);
        out += line;
    }
    if (buf && buf_bytes > 0) {
        snprintf(buf, (size_t)buf_bytes, "%s", out.c_str());
    }
    return NNP_OK;
}
extern "C" int nnp_version(void) { return 102; }
extern "C" int nnp_abi_sizeof(int which)
{
    switch (which) {
    case 0: return (int)sizeof(nnp_nl_params);
    case 1: return (int)sizeof(nnp_tn_model);
    case 2: return (int)sizeof(nnp_prior_params);
    default: return -1;
    }
}

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int block_exclusive_scan(int v, int *total)
{
    __shared__ int warp_sums[SCAN_THREADS / 32];
    __shared__ int block_total;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(NNP_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int w = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
        int winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(NNP_FULL_MASK, winc, o);
            if (lane >= o) winc += t;
        }
        if (lane < SCAN_THREADS / 32) warp_sums[lane] = winc - w;
        if (lane == 31) block_total = winc;
    }
    __syncthreads();
    *total = block_total;
    int result = warp_sums[wid] + inc - v;
    __syncthreads();
    return result;
}

__global__ void scan_tiles(const int32_t *in, int32_t *out, int64_t n, int32_t *tile_totals)
{
    NNP_PDL_SYNC();
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        sum += v[k];
    }
    int total;
    int prefix = block_exclusive_scan(sum, &total);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) out[base + k] = prefix;
        prefix += v[k];
    }
    if (threadIdx.x == 0) tile_totals[blockIdx.x] = total;
}

__global__ void scan_totals(int32_t *tile_totals, int nt)
{
    NNP_PDL_SYNC();
    __shared__ int carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < nt; base += SCAN_THREADS) {
        int idx = base + threadIdx.x;
        int v = idx < nt ? tile_totals[idx] : 0;
        int total;
        int prefix = block_exclusive_scan(v, &total);
        int carry = carry_s;
        if (idx < nt) tile_totals[idx] = carry + prefix;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + total;
        __syncthreads();
    }
}

__global__ void scan_add(int32_t *__restrict__ out, int64_t n, const int32_t *__restrict__ tile_totals)
{
    NNP_PDL_SYNC();
    const int add = tile_totals[blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
        if (base + k < n) out[base + k] += add;
}

}  // namespace

size_t nnp_scan_temp_ints(int64_t n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }

int nnp_exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, int32_t *temp,
                           cudaStream_t stream)
{
    if (n <= 0) return NNP_OK;
    const int nt = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
    nnp_launch((scan_tiles), NNP_GRID(nt), SCAN_THREADS, 0, stream, in, out, n, temp);
    if (nt > 1) {
        nnp_launch((scan_totals), NNP_GRID(1), SCAN_THREADS, 0, stream, temp, nt);
        nnp_launch((scan_add), NNP_GRID(nt), SCAN_THREADS, 0, stream, out, n, temp);
    }
    NNP_CHECK_LAUNCH("exclusive_scan");
    return NNP_OK;
}
