// Host worker pool: the file codec's shard reads/writes and the host-buffer
// pipeline's packing of pageable symbols into pinned staging run on it.
// run(n, f) executes f(0..n-1) on the workers and the calling thread and
// rethrows the first failure; several callers may run jobs at once.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pyrit_b200 {

class HostPool {
public:
    HostPool() {
        const unsigned n = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        for (unsigned i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& th : workers_) th.join();
    }
    // f(0..n-1) on the workers and the caller; rethrows the first failure
    void run(std::size_t n, const std::function<void(std::size_t)>& f) {
        if (n == 0) return;
        Job job{&f, n, 0, 0, nullptr};
        std::unique_lock<std::mutex> lk(mu_);
        jobs_.push_back(&job);
        cv_.notify_all();
        // an item is claimed (next++) under the lock and counted as finished
        // only after it ran, so the job outlives every worker touching it
        while (job.next < job.n) {
            const std::size_t i = job.next++;
            lk.unlock();
            execute(job, i);
            lk.lock();
        }
        done_cv_.wait(lk, [&] { return job.finished == job.n; });
        jobs_.erase(std::remove(jobs_.begin(), jobs_.end(), &job), jobs_.end());
        if (job.error) std::rethrow_exception(job.error);
    }

private:
    struct Job {
        const std::function<void(std::size_t)>* f;
        std::size_t n, next, finished;
        std::exception_ptr error;
    };
    // runs item i of job (claimed by the caller) and records completion
    void execute(Job& job, std::size_t i) {
        std::exception_ptr err;
        try {
            (*job.f)(i);
        } catch (...) {
            err = std::current_exception();
        }
        std::lock_guard<std::mutex> lk(mu_);
        if (err && !job.error) job.error = err;
        if (++job.finished == job.n) done_cv_.notify_all();
    }
    void loop() {
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            Job* job = nullptr;
            cv_.wait(lk, [&] {
                if (stop_) return true;
                for (Job* j : jobs_)
                    if (j->next < j->n) {
                        job = j;
                        return true;
                    }
                return false;
            });
            if (stop_) return;
            const std::size_t i = job->next++;
            lk.unlock();
            execute(*job, i);
            lk.lock();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<Job*> jobs_;
    std::vector<std::thread> workers_;
    bool stop_ = false;
};


HostPool& host_pool(); // min(16, hardware threads) - 1 workers + the caller

} // namespace pyrit_b200
