#include "runtime.hpp"

#include <cstdlib>
#include <memory>

namespace fastnn::b200 {

namespace {

int g_default_device() {
    const char* env = std::getenv("FASTNN_DEVICE");
    return env ? std::atoi(env) : 0;
}

struct ThreadContext {
    int device = -1;
    fnl_context* ctx = nullptr;
    ~ThreadContext() {
        if (ctx) fnl_context_destroy(ctx);
    }
};

thread_local ThreadContext t_ctx;
thread_local int t_device = -1;

}  // namespace

void set_device(int device) { t_device = device; }

int current_device() { return t_device >= 0 ? t_device : g_default_device(); }

fnl_context* context() {
    const int dev = current_device();
    if (t_ctx.ctx && t_ctx.device == dev) return t_ctx.ctx;
    if (t_ctx.ctx) {
        fnl_context_destroy(t_ctx.ctx);
        t_ctx.ctx = nullptr;
    }
    fnl_context* c = nullptr;
    check(fnl_context_create(dev, &c));
    t_ctx.ctx = c;
    t_ctx.device = dev;
    return c;
}

}  // namespace fastnn::b200
