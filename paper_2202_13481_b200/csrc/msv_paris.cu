// K4 paris_kernel: batched paris_plan (paris.hpp:329-345), one warp per job.
//
//   knees      knee() per size (profile.hpp:275-280): first batch whose utilization
//              reaches the threshold = first set bit of a warp ballot over the
//              size's utilization row (32 batches per ballot), else b_max;
//   segments   segment_batches (paris.hpp:34-49): lane s owns size s, its first
//              batch is the previous lane's knee + 1 (shuffle), the last size runs
//              to b_max; knees must be nondecreasing in k;
//   ratios     instance_ratios (paris.hpp:64-81): lane s folds Dist(b)/Thr(k,b) and
//              Dist(b) over its segment in batch order (the reference's left fold);
//              the first failing (segment, batch) in reference order wins;
//   counts     instance_counts (paris.hpp:92-105) and pack_plan (paris.hpp:186-262):
//              lane 0, integer first-fit over the job's GPUs, in the reference's
//              order (floors largest-first, remainders by fraction, greedy fill by
//              segment mass).
// Every FP operation is the reference's, in its order, RN without contraction.
#include "msv_device.cuh"

namespace msv {

namespace {

constexpr int kParisWarps = 4;

__global__ void __launch_bounds__(kParisWarps * 32) paris_kernel(const ParisParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * kParisWarps + (threadIdx.x >> 5);
    if (j >= p.n_jobs) return;
    const ParisJobDev J = p.jobs[j];
    msv_paris_out* o = p.out + j;
    const int n = J.n_sizes;
    const int bmax = J.b_max;
    int status = J.pad;  // host-detected failure (e.g. too many sizes)
    int err_k = 0, err_b = 0;
    const double thr_knee = J.knee_threshold;
    if (status == 0 && J.dist_b_max != bmax) status = MSV_VALIDATION;           // paris.hpp:332-333
    if (status == 0 && (!(thr_knee > 0.0) || thr_knee > 1.0)) status = MSV_PARAM;  // profile.hpp:276

    // ---- knees (ballot over the utilization row) ----
    const int my_k = lane < n ? J.sizes[lane] : 0;
    int my_knee = bmax;
    if (status == 0) {
        for (int s = 0; s < n; ++s) {
            const double* urow = p.util + J.row0 + (int64_t)s * bmax;
            int kn = bmax;
            for (int base = 0; base < bmax; base += 32) {
                const int b = base + lane;
                const unsigned bal = __ballot_sync(kFull, b < bmax && urow[b] >= thr_knee);
                if (bal) {
                    kn = base + __ffs(bal);  // batch = index + 1
                    break;
                }
            }
            if (lane == s) my_knee = kn;
        }
    }
    // ---- segments ----
    const int prev = __shfl_up_sync(kFull, my_knee, 1);
    const int first = (lane == 0 ? 0 : prev) + 1;
    const int last = (lane == n - 1) ? bmax : my_knee;
    if (status == 0) {
        const unsigned bad = __ballot_sync(kFull, lane > 0 && lane < n && my_knee < prev);
        if (bad) status = MSV_VALIDATION;  // paris.hpp:42-44
    }
    // ---- ratios: lane s folds its segment in batch order ----
    double ratio = 0.0, mass = 0.0;
    int fail_b = 0;
    if (status == 0 && lane < n) {
        const double* lrow = p.lat + J.row0 + (int64_t)lane * bmax;
        const double* pmf = p.pmf + J.pmf_off;
        for (int b = first; b <= last && b <= J.dist_b_max; ++b) {
            const double thr = 1000.0 / lrow[b - 1];  // throughput_qps (profile.hpp:108)
            if (!(thr > 0.0)) {
                fail_b = b;
                break;
            }
            ratio = ratio + pmf[b - 1] / thr;
            mass = mass + pmf[b - 1];
        }
    }
    if (status == 0) {
        const unsigned bad = __ballot_sync(kFull, fail_b != 0);
        if (bad) {
            const int s = __ffs(bad) - 1;
            status = MSV_VALIDATION;  // paris.hpp:72-75
            err_k = __shfl_sync(kFull, my_k, s);
            err_b = __shfl_sync(kFull, fail_b, s);
        }
    }
    if (lane < MSV_PARIS_MAX_SIZES) {
        o->k[lane] = my_k;
        o->knee[lane] = lane < n ? my_knee : 0;
        o->seg_first[lane] = lane < n ? first : 0;
        o->seg_last[lane] = lane < n ? last : 0;
        o->ratio[lane] = ratio;
        o->segment_mass[lane] = mass;
        o->count[lane] = 0.0;
    }
    // gather the per-size values into lane 0's registers (n <= 8)
    int ks[MSV_PARIS_MAX_SIZES];
    double rs[MSV_PARIS_MAX_SIZES], ms[MSV_PARIS_MAX_SIZES];
#pragma unroll
    for (int s = 0; s < MSV_PARIS_MAX_SIZES; ++s) {
        ks[s] = __shfl_sync(kFull, my_k, s);
        rs[s] = __shfl_sync(kFull, ratio, s);
        ms[s] = __shfl_sync(kFull, mass, s);
    }
    if (lane != 0) return;

    // ---- instance_counts (paris.hpp:92-105) ----
    double cnt[MSV_PARIS_MAX_SIZES] = {};
    double ws = 0.0, norm = 0.0;
    if (status == 0 && J.total_gpcs < 1) status = MSV_PARAM;
    if (status == 0) {
        for (int s = 0; s < n; ++s) {
            if (rs[s] < 0.0) {
                status = MSV_VALIDATION;
                break;
            }
            ws = ws + (double)ks[s] * rs[s];
        }
        if (status == 0 && !(ws > 0.0)) status = MSV_PARAM;
        if (status == 0) {
            norm = (double)J.total_gpcs / ws;
            for (int s = 0; s < n; ++s) cnt[s] = norm * rs[s];
        }
    }
    // ---- pack_plan (paris.hpp:186-262) ----
    int n_inst = 0;
    const int G = J.num_gpus, C = J.gpcs_per_gpu;
    if (status == 0 && (G < 1 || C < 1)) status = MSV_PARAM;
    double budget_real = 0.0;
    if (status == 0) {
        for (int s = 0; s < n; ++s) {
            if (ks[s] < 1 || cnt[s] < 0.0) {
                status = MSV_PARAM;
                break;
            }
            if (cnt[s] > 0.0 && ks[s] > C) {
                status = MSV_INFEASIBLE;
                err_k = ks[s];
                break;
            }
            budget_real = budget_real + (double)ks[s] * cnt[s];
        }
    }
    if (status == 0) {
        long long bl = llround(budget_real);
        const long long cap = (long long)G * (long long)C;
        int budget = (int)(bl < cap ? bl : cap);
        int32_t* rem = p.remaining + J.gpu_off;
        int32_t* per = p.n_per_gpu + J.gpu_off;
        int32_t* slots = p.sizes_flat + J.inst_off;  // [g * C + i] during packing
        for (int g = 0; g < G; ++g) {
            rem[g] = C;
            per[g] = 0;
        }
        auto place = [&](int k) {  // detail::place_instance (paris.hpp:176-184)
            for (int g = 0; g < G; ++g) {
                if (rem[g] >= k) {
                    rem[g] -= k;
                    slots[(int64_t)g * C + per[g]] = k;
                    per[g] += 1;
                    return true;
                }
            }
            return false;
        };
        // floors, largest size first; a failed placement of k fails for every later
        // copy of k (capacities only shrink), and k > budget stays true
        int fk[MSV_PARIS_MAX_SIZES];
        double ff[MSV_PARIS_MAX_SIZES];
        int nf = 0;
        for (int s = 0; s < n; ++s) {
            const int whole = (int)floor(cnt[s] + 1e-9);
            const double frac = cnt[s] - (double)whole;
            if (frac > 1e-9) {
                fk[nf] = ks[s];
                ff[nf] = frac;
                ++nf;
            }
        }
        for (int s = n - 1; s >= 0; --s) {
            const int whole = (int)floor(cnt[s] + 1e-9);
            for (int i = 0; i < whole; ++i) {
                if (ks[s] > budget || !place(ks[s])) break;
                budget -= ks[s];
            }
        }
        // remainders: fraction descending, then k ascending (insertion sort, <= 8)
        for (int a = 1; a < nf; ++a) {
            const int k = fk[a];
            const double f = ff[a];
            int b = a - 1;
            while (b >= 0 && (ff[b] < f || (ff[b] == f && fk[b] > k))) {
                fk[b + 1] = fk[b];
                ff[b + 1] = ff[b];
                --b;
            }
            fk[b + 1] = k;
            ff[b + 1] = f;
        }
        for (int a = 0; a < nf; ++a) {
            if (fk[a] > budget) continue;
            if (place(fk[a])) budget -= fk[a];
        }
        // greedy fill by segment mass, ties toward smaller sizes
        while (budget > 0) {
            int best = 0;
            double wb = 0.0;
            for (int s = 0; s < n; ++s) {
                const int k = ks[s];
                if (k > budget) continue;
                bool fits = false;
                for (int g = 0; g < G && !fits; ++g) fits = rem[g] >= k;
                if (!fits) continue;
                if (best == 0 || ms[s] > wb || (ms[s] == wb && k < best)) {
                    best = k;
                    wb = ms[s];
                }
            }
            if (best == 0) break;
            place(best);
            budget -= best;
        }
        // compact [g * C + i] to the GPU-major flat list (destinations never pass sources)
        for (int g = 0; g < G; ++g)
            for (int i = 0; i < per[g]; ++i) slots[n_inst++] = slots[(int64_t)g * C + i];
    }
    for (int s = 0; s < n && s < MSV_PARIS_MAX_SIZES; ++s) o->count[s] = cnt[s];
    o->status = status;
    o->n_sizes = n;
    o->n_instances = n_inst;
    o->err_k = err_k;
    o->err_b = err_b;
    o->pad = 0;
    o->weighted_sum = ws;
    o->normalizer = norm;
}

}  // namespace

cudaError_t launch_paris(const ParisParams& p, cudaStream_t stream) {
    if (p.n_jobs <= 0) return cudaSuccess;
    const int64_t blocks = (p.n_jobs + kParisWarps - 1) / kParisWarps;
    paris_kernel<<<(unsigned)blocks, kParisWarps * 32, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace msv
