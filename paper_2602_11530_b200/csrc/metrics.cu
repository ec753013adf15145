// metrics.cu — latency-model outputs and metric reduction on the device.
//
//   rows_kernel     ttft / ttfat / qoe / slo / blocking per request
//                   (proj/src/metrics.cpp:34-68); one thread per request so the
//                   QoE areas are summed sequentially in token order, as the
//                   reference does (:45-49) — bit-exact, never a tree sum.
//   segmented sort  TTFTs per replica (CUB segmented sort).
//   summary_kernel  build_report aggregates (:115-153): mean over the sorted
//                   TTFTs (sequential, sorted order), nearest-rank P50/P90/
//                   P95/P99 (:24-31), SLO-violation rate, TTFAT attainment,
//                   throughput (:70-83); one warp per replica.
//   capacity_kernel derive_capacity's fraction rule (engine.cpp:466-470).

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include <cub/device/device_segmented_sort.cuh>

#include "engine.h"

namespace pb {

constexpr unsigned FULLM = 0xffffffffu;

__global__ void capacity_kernel(ReplicaDesc* desc, const ReplicaOut* oout, const int* map,
                                const int* oref, const double* fraction,
                                const long long* biggest, long long* echo, int count) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    int r = map[k];  // replica, and the oracle pre-run it shares
    double f = fraction[r] > 0.0 ? fraction[r] : 1.0;
    double q = __ddiv_rn(__dmul_rn(f, (double)oout[oref[k]].peak), (double)desc[r].ni);
    long long cap = (long long)ceil(q);
    if (cap < biggest[r]) cap = biggest[r];
    echo[r] = cap;
    if (desc[r].policy != kOracle) desc[r].capacity = cap;
}

__global__ void rows_kernel(const int* rid, const MetricParams* params, const int4* spec,
                            const long long* aoff, const RecOut* rec, const PacerHot* ph,
                            const double* bpv, const int* bpk, const ReqState* rs,
                            RowArrays rows, long long total) {
    long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total) return;
    const MetricParams mp = params[rid[g]];
    const RecOut r = rec[g];
    const int4 sp = spec[g];
    // ttft / ttfat (metrics.cpp:34-36)
    double ttft = __dsub_rn(r.first_answer_delivery, r.arrival);
    double ttfat = __dsub_rn(r.first_answer_delivery, r.reasoning_end);
    // qoe (metrics.cpp:38-52)
    double q = 1.0;
    int nd = rs[g].ndel;
    long long n = sp.z;
    if (n >= 1 && nd > 0) {
        const PacerHot p = ph[g];
        const double* bv = bpv + aoff[g];
        const int* bk = bpk + aoff[g];
        double t0 = r.first_answer_delivery;
        double horizon = p.dlast;
        if (horizon > t0) {
            // digests replayed from their breakpoints (engine.h PacerHot)
            double da = 0.0, d = 0.0;
            int j = 0, kn = p.nbp > 0 ? bk[0] : INT_MAX;
            for (int k = 0; k < nd; ++k) {
                if (k == kn) {
                    d = bv[j];
                    ++j;
                    kn = j < p.nbp ? bk[j] : INT_MAX;
                } else {
                    d = __dadd_rn(d, mp.tpot);
                }
                double x = __dsub_rn(horizon, d);
                da = __dadd_rn(da, 0.0 < x ? x : 0.0);
            }
            double ea = 0.0;
            for (long long k = 0; k < n; ++k) {
                double x = __dsub_rn(horizon, __dadd_rn(t0, __dmul_rn((double)k, mp.tpot)));
                ea = __dadd_rn(ea, 0.0 < x ? x : 0.0);
            }
            if (ea > 0.0) q = __ddiv_rn(da, ea);
        }
    }
    // blocking latency (metrics.cpp:58-68)
    double lo = r.reasoning_end, hi = r.first_answer_iter_start, mig = 0.0;
    if (r.nmig) {
        double a = lo < r.mig_start ? r.mig_start : lo;
        double b = r.mig_end < hi ? r.mig_end : hi;
        if (b > a) mig = __dadd_rn(mig, __dsub_rn(b, a));
    }
    double blk = __dsub_rn(__dsub_rn(hi, lo), mig);
    if (!(0.0 < blk)) blk = 0.0;
    rows.ttft[g] = ttft;
    rows.ttfat[g] = ttfat;
    rows.qoe[g] = q;
    rows.blocking[g] = blk;
    rows.slo[g] = q < mp.qoe_threshold ? 1 : 0;
    // per-request TPOT (not a reference output): the answer
    // tokens after the first are delivered over [first delivery, completion]
    // (the last token is delivered at the finishing iteration's end,
    // engine.cpp:320-337)
    rows.tpot[g] = sp.z > 1 ? __ddiv_rn(__dsub_rn(r.completion, r.first_answer_delivery),
                                        (double)(sp.z - 1))
                            : 0.0;
}

__device__ __forceinline__ double nearest_rank(const double* v, long long n, double pct) {
    long long rank = (long long)ceil(__dmul_rn(pct, (double)n));
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return v[rank - 1];
}

__global__ void summary_kernel(const MetricParams* params, const ReplicaDesc* desc,
                               const ReplicaOut* out, const int4* spec, const RecOut* rec,
                               RowArrays rows, const long long* echo, DevSummary* sum,
                               int n_rep) {
    int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (r >= n_rep) return;
    const MetricParams mp = params[r];
    const ReplicaOut o = out[r];
    const long long base = mp.req_base, n = mp.n;
    DevSummary s;
    s.ttft_mean = s.ttft_p50 = s.ttft_p90 = s.ttft_p95 = s.ttft_p99 = 0.0;
    s.slo_rate = s.ttfat_attain = s.throughput = 0.0;
    s.capacity = echo[r];
    s.requests = n;
    s.req_iters = o.req_iters;
    s.answer_tokens = o.answer_tokens;
    s.events = o.events;
    s.plans = o.plans;
    s.visits = o.visits;
    s.health = o.health_checks;
    s.slo_violations = 0;
    s.adm_rounds = o.adm_rounds;
    s.adm_slow = o.adm_slow;
    s.status = o.status;
    s.pad = 0;
    s.tpot_mean = 0.0;
    s.tpot_requests = 0;
    if (o.status == 0 && n > 0) {
        long long viol = 0, ok = 0, tokens = 0, ntp = 0;
        double tsum = 0.0;
        double first = rec[base].arrival, last = rec[base].completion;
        for (long long k = lane; k < n; k += 32) {
            long long g = base + k;
            viol += rows.slo[g];
            ok += rows.ttfat[g] <= mp.ttfat_target ? 1 : 0;
            int4 sp = spec[g];
            tokens += (long long)sp.y + sp.z;
            if (sp.z > 1) {
                tsum = __dadd_rn(tsum, rows.tpot[g]);
                ++ntp;
            }
            double a = rec[g].arrival, c = rec[g].completion;
            first = a < first ? a : first;
            last = last < c ? c : last;
        }
        for (int off = 16; off; off >>= 1) {
            viol += __shfl_xor_sync(FULLM, viol, off);
            ok += __shfl_xor_sync(FULLM, ok, off);
            tokens += __shfl_xor_sync(FULLM, tokens, off);
            ntp += __shfl_xor_sync(FULLM, ntp, off);
            tsum = __dadd_rn(tsum, __shfl_xor_sync(FULLM, tsum, off));
            double f2 = __shfl_xor_sync(FULLM, first, off);
            double l2 = __shfl_xor_sync(FULLM, last, off);
            first = f2 < first ? f2 : first;
            last = last < l2 ? l2 : last;
        }
        if (lane == 0) {
            const double* srt = rows.ttft_sorted + base;
            double acc = 0.0;  // sorted-order sequential sum (metrics.cpp:139-143)
            for (long long k = 0; k < n; ++k) acc = __dadd_rn(acc, srt[k]);
            double dn = (double)n;
            s.ttft_mean = __ddiv_rn(acc, dn);
            s.ttft_p50 = nearest_rank(srt, n, 0.50);
            s.ttft_p90 = nearest_rank(srt, n, 0.90);
            s.ttft_p95 = nearest_rank(srt, n, 0.95);
            s.ttft_p99 = nearest_rank(srt, n, 0.99);
            s.slo_rate = __ddiv_rn((double)viol, dn);
            s.ttfat_attain = __ddiv_rn((double)ok, dn);
            s.slo_violations = viol;
            double span = __dsub_rn(last, first);
            s.throughput = span <= 0.0 ? 0.0 : __ddiv_rn((double)tokens, span);
            s.tpot_requests = ntp;
            s.tpot_mean = ntp > 0 ? __ddiv_rn(tsum, (double)ntp) : 0.0;
        }
    }
    if (lane == 0) sum[r] = s;
}

// Per-group TTFT histogram + SLO counters over all requests of the group's
// replicas (the sweep's device-side reduction; merged across GPUs by NCCL).
// Counters are privatised per CTA in shared memory (32-bit) and flushed once
// per CTA with 64-bit global atomics on the non-zero bins only; a batch's
// requests are grouped by replica, so a CTA's requests fall in few groups and
// the flush is a few hundred atomics instead of three per request.
__device__ __forceinline__ int ttft_bin(double t) {
    if (!(t >= 1e-4)) return 0;
    if (t >= 1e5) return kHistBins + 1;
    return 1 + min(kHistBins - 1, (int)((log10(t) + 4.0) * (kHistBins / 9.0)));
}

__global__ void hist_smem_kernel(const int* rid, const int* group, RowArrays rows,
                                 const ReplicaOut* out, long long total, int n_groups,
                                 unsigned long long* hist, unsigned long long* slo) {
    extern __shared__ unsigned sh[];  // [n_groups][kHistBins + 2] then [n_groups][2]
    const int nh = n_groups * (kHistBins + 2), ns = 2 * n_groups;
    for (int k = threadIdx.x; k < nh + ns; k += blockDim.x) sh[k] = 0u;
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
        const int r = rid[g];
        if (out[r].status != 0) continue;
        const int grp = group[r];
        atomicAdd(&sh[grp * (kHistBins + 2) + ttft_bin(rows.ttft[g])], 1u);
        if (rows.slo[g]) atomicAdd(&sh[nh + 2 * grp], 1u);
        atomicAdd(&sh[nh + 2 * grp + 1], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nh; k += blockDim.x)
        if (sh[k]) atomicAdd(&hist[k], (unsigned long long)sh[k]);
    for (int k = threadIdx.x; k < ns; k += blockDim.x)
        if (sh[nh + k]) atomicAdd(&slo[k], (unsigned long long)sh[nh + k]);
}

// Fallback for group counts whose counters do not fit in shared memory.
__global__ void hist_kernel(const int* rid, const int* group, RowArrays rows,
                            const ReplicaOut* out, long long total, unsigned long long* hist,
                            unsigned long long* slo) {
    long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total) return;
    const int r = rid[g];
    if (out[r].status != 0) return;
    const int grp = group[r];
    atomicAdd(&hist[(long long)grp * (kHistBins + 2) + ttft_bin(rows.ttft[g])], 1ull);
    atomicAdd(&slo[2 * grp], (unsigned long long)rows.slo[g]);
    atomicAdd(&slo[2 * grp + 1], 1ull);
}

int launch_histograms(const int* rid, const int* group, const RowArrays rows,
                      const ReplicaOut* out, long long total, int n_groups,
                      unsigned long long* hist, unsigned long long* slo, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * n_groups * (kHistBins + 2), st);
    cudaMemsetAsync(slo, 0, sizeof(unsigned long long) * n_groups * 2, st);
    if (total > 0) {
        const size_t smem = sizeof(unsigned) * (size_t)n_groups * (kHistBins + 4);
        if (smem <= 96 * 1024) {
            // opt in above 48 KB (a per-device function attribute: set on
            // every launch, the batch may live on any device)
            cudaFuncSetAttribute(hist_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 96 * 1024);
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const long long want = (total + 1023) / 1024;
            const int blocks = (int)std::min<long long>(want, 2ll * sms);
            hist_smem_kernel<<<blocks, 512, smem, st>>>(rid, group, rows, out, total, n_groups,
                                                       hist, slo);
        } else {
            hist_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(rid, group, rows, out,
                                                                         total, hist, slo);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_capacity(ReplicaDesc* desc, const ReplicaOut* oracle_out, const int* map,
                    const int* oref, const double* fraction, const long long* biggest,
                    long long* echo, int count, void* stream) {
    if (count <= 0) return 0;
    capacity_kernel<<<(count + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        desc, oracle_out, map, oref, fraction, biggest, echo, count);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_metrics(const Arena& a, const MetricParams* params, const long long* seg,
                   const int* rid, long long total, int n_rep, RowArrays rows,
                   DevSummary* out, const long long* echo_capacity, void* sort_tmp,
                   size_t* sort_tmp_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    // CUB's segmented sort counts items in int; Batch::build rejects larger
    // batches (engine_host.cpp), this is the backstop
    if (total > (long long)INT_MAX) return 4;
    if (sort_tmp == nullptr) {  // size query
        size_t bytes = 0;
        cudaError_t e = cub::DeviceSegmentedSort::SortKeys(
            nullptr, bytes, rows.ttft, rows.ttft_sorted, (int)(total > 0 ? total : 1), n_rep,
            seg, seg + 1, st);
        *sort_tmp_bytes = bytes;
        return e == cudaSuccess ? 0 : 1;
    }
    if (total > 0) {
        rows_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
            rid, params, a.spec, a.aoff, a.rec, a.ph, a.bpv, a.bpk, a.rs, rows, total);
        size_t bytes = *sort_tmp_bytes;
        if (cub::DeviceSegmentedSort::SortKeys(sort_tmp, bytes, rows.ttft, rows.ttft_sorted,
                                               (int)total, n_rep, seg, seg + 1,
                                               st) != cudaSuccess)
            return 2;
    }
    summary_kernel<<<(n_rep * 32 + 127) / 128, 128, 0, st>>>(params, a.desc, a.out, a.spec,
                                                              a.rec, rows, echo_capacity, out,
                                                              n_rep);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace pb
