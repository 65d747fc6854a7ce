// Host-side system features of ParaGAN (PAPER.md:221-233 [Sec. 4.1]):
//  * the congestion-aware prefetcher: reader threads fill a bounded queue of batches from sample
//    shards; a sliding window of read latencies scales the number of active readers and the queue
//    depth up when the window mean exceeds a threshold and releases them when it falls back (P:231
//    "If the current latency over the window exceeds the threshold, ParaGAN will increase the number
//    of threads and buffer for pre-fetching and pre-processing; once the latency falls below the
//    threshold, it releases the resources");
//  * the asynchronous checkpoint writer lives in engine.cu (it needs the engine's buffers); its file
//    format helpers are here.
// Pure host C++ (std::thread); no CUDA calls, so it also runs on a machine without a GPU.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/paragan.h"
#include "host_io.h"

namespace pg {

uint64_t fnv1a64(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace pg

namespace {

constexpr char kShardMagic[8] = {'P', 'G', 'S', 'H', 'A', 'R', 'D', '1'};

struct Shard {
  std::string path;
  long long n = 0;
};

}  // namespace

struct paragan_prefetcher {
  paragan_prefetch_config cfg{};
  std::vector<Shard> shards;
  long long total = 0;                  // samples over all shards
  size_t sample_floats = 0;
  // batch queue: index -> (images, labels); next() hands them out in index order
  std::mutex mu;
  std::condition_variable cv_ready, cv_space, cv_work;
  std::map<long long, std::pair<std::vector<float>, std::vector<int32_t>>> ready;
  long long next_issue = 0, next_out = 0;
  int active = 1, depth = 2;            // current readers / queue depth (the tuned resources)
  int busy = 0;
  bool stop = false;
  std::string error;
  // latency window (ms per batch read)
  std::deque<double> window;
  double window_sum = 0.0;
  long long reads = 0, scale_ups = 0, scale_downs = 0;
  std::atomic<float> inject_ms{0.0f};
  std::vector<std::thread> threads;

  // samples [start, start + count) (cyclic over the shards in order): one open + two reads per shard run
  bool read_range(long long start, int count, float* img, int32_t* label) {
    int done = 0;
    while (done < count) {
      long long idx = (start + done) % total;
      for (const Shard& s : shards) {
        if (idx >= s.n) {
          idx -= s.n;
          continue;
        }
        const int run = (int)std::min<long long>(count - done, s.n - idx);
        FILE* f = std::fopen(s.path.c_str(), "rb");
        if (!f) return false;
        const long long hdr = 8 + 4 * 4;
        bool ok = std::fseek(f, (long)(hdr + idx * 4), SEEK_SET) == 0 &&
                  std::fread(label + done, 4, (size_t)run, f) == (size_t)run &&
                  std::fseek(f, (long)(hdr + s.n * 4 + idx * (long long)sample_floats * 4), SEEK_SET) == 0 &&
                  std::fread(img + (size_t)done * sample_floats, sizeof(float), sample_floats * run, f) ==
                      sample_floats * run;
        std::fclose(f);
        if (!ok) return false;
        done += run;
        break;
      }
    }
    return true;
  }

  // controller: called with mu held after every read
  void tune(double ms) {
    window.push_back(ms);
    window_sum += ms;
    if ((int)window.size() > cfg.window) {
      window_sum -= window.front();
      window.pop_front();
    }
    ++reads;
    if ((int)window.size() < cfg.window || reads % cfg.window) return;   // decide once per full window
    const double mean = window_sum / window.size();
    if (mean > cfg.latency_threshold_ms) {
      if (active < cfg.max_workers || depth < cfg.max_depth) ++scale_ups;
      active = std::min(active + 1, cfg.max_workers);
      depth = std::min(depth * 2, cfg.max_depth);
    } else if (mean < 0.5 * cfg.latency_threshold_ms) {
      if (active > cfg.min_workers || depth > cfg.min_depth) ++scale_downs;
      active = std::max(active - 1, cfg.min_workers);
      depth = std::max(depth / 2, cfg.min_depth);
    }
    cv_work.notify_all();
    cv_space.notify_all();
  }

  void worker(int id) {
    const int B = cfg.batch;
    for (;;) {
      long long bi;
      {
        std::unique_lock<std::mutex> lk(mu);
        // a reader works only while it is among the active ones and the queue has room
        cv_work.wait(lk, [&] {
          return stop || (id < active && next_issue - next_out < depth);
        });
        if (stop) return;
        bi = next_issue++;
        ++busy;
      }
      std::vector<float> img((size_t)B * sample_floats);
      std::vector<int32_t> lab(B);
      const auto t0 = std::chrono::steady_clock::now();
      const float extra = inject_ms.load();
      if (extra > 0.0f) std::this_thread::sleep_for(std::chrono::microseconds((long long)(extra * 1000.0f)));
      const bool ok = read_range(bi * B, B, img.data(), lab.data());
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      {
        std::lock_guard<std::mutex> lk(mu);
        --busy;
        if (!ok && error.empty()) error = "prefetch: read failed for batch " + std::to_string(bi);
        ready.emplace(bi, std::make_pair(std::move(img), std::move(lab)));
        tune(ms);
      }
      cv_ready.notify_all();
    }
  }
};

extern "C" {

paragan_status paragan_shard_write(const char* path, const float* images, const int32_t* labels, int32_t n,
                                   int32_t c, int32_t h, int32_t w) {
  if (!path || !images || !labels || n < 1 || c < 1 || h < 1 || w < 1) return PARAGAN_ERR_INVALID_ARG;
  FILE* f = std::fopen(path, "wb");
  if (!f) return PARAGAN_ERR_IO;
  const int32_t hdr[4] = {n, c, h, w};
  const size_t per = (size_t)c * h * w;
  bool ok = std::fwrite(kShardMagic, 1, 8, f) == 8 && std::fwrite(hdr, 4, 4, f) == 4 &&
            std::fwrite(labels, 4, (size_t)n, f) == (size_t)n &&
            std::fwrite(images, sizeof(float), per * n, f) == per * n;
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PARAGAN_OK : PARAGAN_ERR_IO;
}

paragan_status paragan_prefetch_create(const paragan_prefetch_config* cfg, const char* const* shard_paths,
                                       int32_t n_shards, paragan_prefetcher** out) {
  if (!cfg || !shard_paths || n_shards < 1 || !out) return PARAGAN_ERR_INVALID_ARG;
  if (cfg->batch < 1 || cfg->min_workers < 1 || cfg->max_workers < cfg->min_workers || cfg->min_depth < 1 ||
      cfg->max_depth < cfg->min_depth || cfg->window < 1 || !(cfg->latency_threshold_ms > 0.0f))
    return PARAGAN_ERR_CONFIG;
  auto* p = new paragan_prefetcher;
  p->cfg = *cfg;
  p->sample_floats = (size_t)cfg->channels * cfg->height * cfg->width;
  for (int i = 0; i < n_shards; ++i) {
    FILE* f = std::fopen(shard_paths[i], "rb");
    if (!f) {
      delete p;
      return PARAGAN_ERR_IO;
    }
    char magic[8];
    int32_t hdr[4];
    const bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kShardMagic, 8) == 0 &&
                    std::fread(hdr, 4, 4, f) == 4 && hdr[1] == cfg->channels && hdr[2] == cfg->height &&
                    hdr[3] == cfg->width && hdr[0] > 0;
    std::fclose(f);
    if (!ok) {
      delete p;
      return PARAGAN_ERR_IO;
    }
    p->shards.push_back(Shard{shard_paths[i], hdr[0]});
    p->total += hdr[0];
  }
  p->active = cfg->min_workers;
  p->depth = cfg->min_depth;
  p->inject_ms = cfg->inject_latency_ms;
  for (int i = 0; i < cfg->max_workers; ++i) p->threads.emplace_back(&paragan_prefetcher::worker, p, i);
  *out = p;
  return PARAGAN_OK;
}

paragan_status paragan_prefetch_next(paragan_prefetcher* p, float* images, int32_t* labels) {
  if (!p || !images || !labels) return PARAGAN_ERR_INVALID_ARG;
  std::pair<std::vector<float>, std::vector<int32_t>> b;
  {
    std::unique_lock<std::mutex> lk(p->mu);
    p->cv_ready.wait(lk, [&] { return p->ready.count(p->next_out) > 0 || !p->error.empty(); });
    if (!p->error.empty()) return PARAGAN_ERR_IO;
    auto it = p->ready.find(p->next_out);
    b = std::move(it->second);
    p->ready.erase(it);
    ++p->next_out;
  }
  p->cv_work.notify_all();
  std::memcpy(images, b.first.data(), b.first.size() * sizeof(float));
  std::memcpy(labels, b.second.data(), b.second.size() * sizeof(int32_t));
  return PARAGAN_OK;
}

paragan_status paragan_prefetch_set_latency(paragan_prefetcher* p, float inject_ms) {
  if (!p || inject_ms < 0.0f) return PARAGAN_ERR_INVALID_ARG;
  p->inject_ms = inject_ms;
  return PARAGAN_OK;
}

paragan_status paragan_prefetch_get_stats(paragan_prefetcher* p, paragan_prefetch_stats* out) {
  if (!p || !out) return PARAGAN_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(p->mu);
  out->active_workers = p->active;
  out->depth = p->depth;
  out->queued = (int32_t)p->ready.size();
  out->window_mean_ms = p->window.empty() ? 0.0f : (float)(p->window_sum / p->window.size());
  out->batches_read = p->reads;
  out->scale_ups = p->scale_ups;
  out->scale_downs = p->scale_downs;
  return PARAGAN_OK;
}

paragan_status paragan_prefetch_destroy(paragan_prefetcher* p) {
  if (!p) return PARAGAN_ERR_INVALID_ARG;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->stop = true;
  }
  p->cv_work.notify_all();
  for (auto& t : p->threads) t.join();
  delete p;
  return PARAGAN_OK;
}

}  // extern "C"
