// Stream-ordered caching device allocator behind the reference's MemoryManager API
// (minml/memory.py:86-347).  Policies and every counter follow the reference exactly:
//   native            grant == request; each free returns the block to the system
//   caching           <=512 B -> 512 B bin, else next power of two; freed blocks are cached
//                     and reused only on an exact bin match (memory.py:243-288)
//   split_restricted  a cached block no larger than `threshold` may be carved: grant the
//                     request rounded up to 512 B, the remainder re-enters the cache unless
//                     it is below 512 B (then it is absorbed) (memory.py:291-334)
// Device specifics the reference has no notion of:
//   * all allocations and frees are ordered on the compute stream, so a freed block can be
//     handed out again immediately without synchronisation;
//   * a block recorded on another stream (NCCL's comm stream) is parked behind a CUDA event
//     at free time and only re-enters the cache once that event has completed;
//   * pools: while a CUDA graph is being captured, allocations come from (and frees return
//     to) a private pool, so eager work between replays can never reuse graph memory;
//   * system memory is tracked per cudaMalloc segment; split pieces keep their segment
//     alive and the segment is cudaFree'd once all of its pieces have been flushed.
// `simulate` runs the identical bookkeeping with fake addresses (CPU tests, no device).
#include <algorithm>
#include <deque>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>
#include "common.cuh"

namespace pb {

static const uint64_t kFloor = 512;
static const uint64_t kGran = 512;

uint64_t bin_size(uint64_t n) {
  if (n <= kFloor) return kFloor;
  uint64_t b = 1;
  while (b < n) b <<= 1;
  return b;
}
uint64_t round_up(uint64_t n) { return (n + kGran - 1) / kGran * kGran; }

struct Segment {
  uint64_t base, size;
  int pieces;  // live blocks + cache entries carved from this segment
};

struct Entry {  // a cached (free) piece
  uint64_t ptr;
  int64_t seg;
  cudaEvent_t ready;  // null = reusable now
};

struct Block {
  uint64_t ptr, requested, granted;
  int64_t seg;
  int32_t op, pool;
  uint32_t streams;  // bitmask of extra streams that used the block
};

class Manager {
 public:
  Manager(int policy, uint64_t threshold, uint64_t capacity, bool simulate)
      : policy_(policy), threshold_(threshold), capacity_(capacity), simulate_(simulate) {}

  ~Manager() { flush_all(true); }

  int alloc(uint64_t nbytes, int32_t op, pb_mm_block* out) {
    std::lock_guard<std::mutex> lk(mu_);
    if (nbytes == 0) return fail(PB_ERR_ALLOC, "allocation size must be positive, got 0");
    uint64_t granted = 0, ptr = 0;
    int64_t seg = -1;
    int rc = acquire(nbytes, &granted, &ptr, &seg);
    if (rc) return rc;
    uint64_t id = ++next_id_;
    live_[id] = Block{ptr, nbytes, granted, seg, op, pool_, 0};
    live_req_ += nbytes;
    live_granted_ += granted;
    peak_granted_ = std::max(peak_granted_, live_granted_);
    peak_internal_ = std::max(peak_internal_, live_granted_ - live_req_);
    if (requests_.size() < (1u << 22)) requests_.push_back(nbytes);
    out->id = id;
    out->ptr = ptr;
    out->requested_bytes = nbytes;
    out->granted_bytes = granted;
    out->bin_size = granted;
    out->op_tag = op;
    out->pool = pool_;
    return PB_OK;
  }

  int free(uint64_t id) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = live_.find(id);
    if (it == live_.end()) return fail(PB_ERR_ALLOC, "free of unknown or already-freed block " + std::to_string(id));
    Block b = it->second;
    live_.erase(it);
    live_req_ -= b.requested;
    live_granted_ -= b.granted;
    cudaEvent_t ev = nullptr;
    if (b.streams && !simulate_ && b.pool == 0) {
      // the block may still be used by another stream: park it behind one event that
      // completes after that stream's work queued so far.  Used on both side streams: the
      // comm stream first waits for the copy stream's work, then records the event.
      // (Graph-capture pools skip this: an event recorded inside a capture cannot be
      // queried, and a recorded step joins its side streams before it ends.)
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      const bool on_comm = b.streams & 2u, on_copy = b.streams & 4u;
      if (on_comm && on_copy) {
        cudaEvent_t j = nullptr;
        cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
        cudaEventRecord(j, copy_stream());
        cudaStreamWaitEvent(comm_stream(), j, 0);
        cudaEventDestroy(j);
      }
      cudaEventRecord(ev, on_comm ? comm_stream() : copy_stream());
    }
    if (policy_ == PB_POLICY_NATIVE) {
      ++free_count_;
      release_piece(b.seg, ev);
      return PB_OK;
    }
    push(b.pool, b.granted, Entry{b.ptr, b.seg, ev});
    return PB_OK;
  }

  int record_stream(uint64_t id, int stream) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = live_.find(id);
    if (it == live_.end()) return fail(PB_ERR_ALLOC, "record_stream on unknown block");
    if (stream > 0 && stream < 3) it->second.streams |= (1u << stream);
    return PB_OK;
  }

  void stats(pb_mm_stats* s) {
    std::lock_guard<std::mutex> lk(mu_);
    s->live_bytes_requested = live_req_;
    s->live_bytes_granted = live_granted_;
    s->peak_granted = peak_granted_;
    s->cache_bytes = cache_total_;
    s->alloc_count = alloc_count_;
    s->free_count = free_count_;
    s->internal_fragmentation = live_granted_ - live_req_;
    s->peak_internal_fragmentation = peak_internal_;
    s->live_blocks = live_.size();
    s->external_fragmentation_ratio = external_ratio();
  }

  uint64_t flush() {
    std::lock_guard<std::mutex> lk(mu_);
    return flush_all(false);
  }

  void set_pool(int pool) {
    std::lock_guard<std::mutex> lk(mu_);
    pool_ = pool;
  }

 private:
  typedef std::map<uint64_t, std::deque<Entry>> Cache;

  Cache& cache(int pool) { return caches_[pool]; }

  void push(int pool, uint64_t size, const Entry& e) {
    cache(pool)[size].push_back(e);
    cache_total_ += size;
  }

  bool ready(Entry& e) {
    if (!e.ready) return true;
    if (cudaEventQuery(e.ready) == cudaSuccess) {
      cudaEventDestroy(e.ready);
      e.ready = nullptr;
      return true;
    }
    cudaGetLastError();
    return false;
  }

  // pop the oldest reusable entry of exactly `size` from the current pool
  bool pop(uint64_t size, Entry* out) {
    Cache& c = cache(pool_);
    auto it = c.find(size);
    if (it == c.end()) return false;
    auto& dq = it->second;
    for (auto e = dq.begin(); e != dq.end(); ++e) {
      if (ready(*e)) {
        *out = *e;
        dq.erase(e);
        cache_total_ -= size;
        if (dq.empty()) c.erase(it);
        return true;
      }
    }
    return false;
  }

  int acquire(uint64_t nbytes, uint64_t* granted, uint64_t* ptr, int64_t* seg) {
    if (policy_ == PB_POLICY_NATIVE) {
      *granted = nbytes;
      return system_alloc(nbytes, ptr, seg);
    }
    if (policy_ == PB_POLICY_SPLIT) {
      uint64_t tight = round_up(nbytes);
      Cache& c = cache(pool_);
      // smallest cached size in [tight, threshold] with a reusable entry
      for (auto it = c.lower_bound(tight); it != c.end() && it->first <= threshold_; ++it) {
        Entry e;
        uint64_t best = it->first;
        if (!pop(best, &e)) continue;
        uint64_t rem = best - tight;
        if (rem >= kFloor) {
          segs_[e.seg].pieces += 1;
          push(pool_, rem, Entry{e.ptr + tight, e.seg, nullptr});
          *granted = tight;
        } else {
          *granted = best;
        }
        *ptr = e.ptr;
        *seg = e.seg;
        return PB_OK;
      }
    }
    uint64_t b = bin_size(nbytes);
    Entry e;
    if (pop(b, &e)) {
      *granted = b;
      *ptr = e.ptr;
      *seg = e.seg;
      return PB_OK;
    }
    *granted = b;
    return system_alloc(b, ptr, seg);
  }

  int system_alloc(uint64_t bytes, uint64_t* ptr, int64_t* seg) {
    if (capacity_) {
      if (live_granted_ + cache_total_ + bytes > capacity_) flush_all(false);
      if (live_granted_ + bytes > capacity_)
        return fail(PB_ERR_OOM, "request for " + std::to_string(bytes) + " bytes exceeds capacity " +
                                    std::to_string(capacity_) + " (" + std::to_string(live_granted_) + " live)");
    }
    uint64_t base;
    if (simulate_) {
      base = fake_next_;
      fake_next_ += (bytes + 255) / 256 * 256;
    } else {
      void* p = nullptr;
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        flush_all(false);  // give cached memory back to the driver and retry once
        e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(PB_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed after a cache flush");
        }
      }
      base = (uint64_t)(uintptr_t)p;
    }
    ++alloc_count_;
    int64_t id = next_seg_++;
    segs_[id] = Segment{base, bytes, 1};
    *ptr = base;
    *seg = id;
    return PB_OK;
  }

  void release_piece(int64_t seg, cudaEvent_t ev) {
    auto it = segs_.find(seg);
    if (it == segs_.end()) return;
    if (--it->second.pieces == 0) {
      if (!simulate_) {
        if (ev) cudaEventSynchronize(ev);
        cudaFree((void*)(uintptr_t)it->second.base);
      }
      segs_.erase(it);
    }
    if (ev) cudaEventDestroy(ev);
  }

  uint64_t flush_all(bool everything) {
    uint64_t released = 0;
    for (auto& pc : caches_) {
      // private pools hold addresses recorded into CUDA graphs: only the destructor frees them
      if (pc.first != 0 && !everything) continue;
      for (auto& kv : pc.second) {
        for (auto& e : kv.second) {
          ++released;
          cache_total_ -= kv.first;
          release_piece(e.seg, e.ready);
        }
      }
      pc.second.clear();
    }
    free_count_ += released;
    return released;
  }

  bool can_serve(uint64_t cached, uint64_t probe) const {
    if (policy_ == PB_POLICY_SPLIT && cached <= threshold_ && cached >= round_up(probe)) return true;
    if (policy_ == PB_POLICY_NATIVE) return false;
    return cached == bin_size(probe);
  }

  double external_ratio() {
    if (cache_total_ == 0 || requests_.empty()) return 0.0;
    std::vector<uint64_t> v(requests_);
    size_t n = v.size();
    std::nth_element(v.begin(), v.begin() + n / 2, v.end());
    double med = (double)v[n / 2];
    if (n % 2 == 0) {
      uint64_t lo = *std::max_element(v.begin(), v.begin() + n / 2);
      med = ((double)lo + (double)v[n / 2]) / 2.0;
    }
    uint64_t probe = (uint64_t)med;  // int(statistics.median(...)) truncates
    uint64_t unusable = 0;
    for (auto& pc : caches_)
      for (auto& kv : pc.second)
        if (!kv.second.empty() && !can_serve(kv.first, probe)) unusable += kv.first * kv.second.size();
    return (double)unusable / (double)cache_total_;
  }

  std::mutex mu_;
  int policy_;
  uint64_t threshold_, capacity_;
  bool simulate_;
  int pool_ = 0;
  std::map<int, Cache> caches_;
  std::unordered_map<uint64_t, Block> live_;
  std::unordered_map<int64_t, Segment> segs_;
  std::vector<uint64_t> requests_;
  uint64_t next_id_ = 0, fake_next_ = 1ull << 40;
  int64_t next_seg_ = 0;
  uint64_t live_req_ = 0, live_granted_ = 0, peak_granted_ = 0, peak_internal_ = 0;
  uint64_t cache_total_ = 0, alloc_count_ = 0, free_count_ = 0;
};

}  // namespace pb

using namespace pb;

extern "C" {

uint64_t pb_bin_size(uint64_t n) { return bin_size(n); }
uint64_t pb_round_up(uint64_t n) { return round_up(n); }

void* pb_mm_create(int policy, uint64_t threshold, uint64_t capacity, int simulate) {
  if (policy < 0 || policy > 2) {
    set_error("unknown allocator policy");
    return nullptr;
  }
  return new Manager(policy, threshold, capacity, simulate != 0);
}

void pb_mm_destroy(void* mm) { delete (Manager*)mm; }

int pb_mm_alloc(void* mm, uint64_t nbytes, int32_t op_tag, pb_mm_block* out) {
  return ((Manager*)mm)->alloc(nbytes, op_tag, out);
}

int pb_mm_free(void* mm, uint64_t id) { return ((Manager*)mm)->free(id); }

int pb_mm_record_stream(void* mm, uint64_t id, int stream) { return ((Manager*)mm)->record_stream(id, stream); }

int pb_mm_stats_get(void* mm, pb_mm_stats* out) {
  ((Manager*)mm)->stats(out);
  return PB_OK;
}

uint64_t pb_mm_flush(void* mm) { return ((Manager*)mm)->flush(); }

int pb_mm_pool(void* mm, int pool) {
  ((Manager*)mm)->set_pool(pool);
  return PB_OK;
}

}  // extern "C"
