// sp_torch.cpp -- the PyTorch C++ extension over the C-ABI (include/sparrow.h).
//
// Registers the hot calls as torch operators (torch.ops.sparrow.*): tensor
// checks (device, dtype, shape, contiguity) in C++, the current CUDA stream
// from ATen, then the C-ABI entry point; a failing status raises with
// sp_last_error().  The entry points are resolved with dlsym from the very
// libsparrow.so the Python package loaded (sparrow::bind(path), called by
// paper_2305_04180_b200._lib), so a variant library selected with
// SPARROW_LIB_PATH is the one both bindings drive.
//
//   sparrow::bind(str lib_path)                  -> ()
//   sparrow::env_step(int handle, Tensor actions, Tensor(a!) states,
//                     Tensor(b!) store_states, Tensor(c!) rewards,
//                     Tensor(d!) dones, Tensor(e!) truncated,
//                     Tensor(f!) events)         -> ()   (vecenv.py:94-116)
//   sparrow::rb_append(int handle, Tensor s, Tensor a, Tensor r, Tensor s2,
//                      Tensor d)                 -> ()   (replay.py:48-67)
#include <dlfcn.h>
#include <torch/library.h>
#include <ATen/ATen.h>
#include <c10/cuda/CUDAStream.h>

#include <string>

#include "../../include/sparrow.h"

namespace {

struct Api {
  void* lib = nullptr;
  decltype(&sp_env_step) env_step = nullptr;
  decltype(&sp_rb_append) rb_append = nullptr;
  decltype(&sp_last_error) last_error = nullptr;
};
Api g_api;

void bind(std::string path) {
  void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_NOLOAD);  // the instance already loaded
  if (!h) h = dlopen(path.c_str(), RTLD_NOW);
  TORCH_CHECK(h, "sparrow: cannot open ", path, ": ", dlerror());
  Api a;
  a.lib = h;
  a.env_step = (decltype(&sp_env_step))dlsym(h, "sp_env_step");
  a.rb_append = (decltype(&sp_rb_append))dlsym(h, "sp_rb_append");
  a.last_error = (decltype(&sp_last_error))dlsym(h, "sp_last_error");
  TORCH_CHECK(a.env_step && a.rb_append && a.last_error, "sparrow: ", path,
              " lacks the C-ABI entry points");
  g_api = a;
}

// The status only: the Python layer reads sp_last_error() itself (through the
// same library) and maps the status to the reference's exception classes.
void check_rc(int rc, const char* what) {
  TORCH_CHECK(rc == SP_OK, "sparrow ", what, " failed (status ", rc, ")");
}

void need(const at::Tensor& t, at::ScalarType dt, const char* name, const at::Device& dev) {
  TORCH_CHECK(t.device() == dev, "sparrow: ", name, " must be on ", dev);
  TORCH_CHECK(t.scalar_type() == dt, "sparrow: ", name, " must be ", dt, ", got ", t.scalar_type());
  TORCH_CHECK(t.is_contiguous(), "sparrow: ", name, " must be contiguous");
}

void env_step(int64_t handle, const at::Tensor& actions, at::Tensor states,
              at::Tensor store_states, at::Tensor rewards, at::Tensor dones,
              at::Tensor truncated, at::Tensor events) {
  TORCH_CHECK(g_api.env_step, "sparrow: call sparrow::bind first");
  const at::Device dev = actions.device();
  TORCH_CHECK(dev.is_cuda(), "sparrow: actions must be a CUDA tensor");
  const int64_t n = actions.numel();
  need(actions, at::kLong, "actions", dev);
  need(states, at::kFloat, "states", dev);
  need(store_states, at::kFloat, "store_states", dev);
  need(rewards, at::kDouble, "rewards", dev);
  need(dones, at::kBool, "dones", dev);
  need(truncated, at::kBool, "truncated", dev);
  need(events, at::kChar, "events", dev);
  TORCH_CHECK(states.dim() == 2 && states.size(0) == n && store_states.sizes() == states.sizes(),
              "sparrow: states / store_states must be (N, 5+R)");
  TORCH_CHECK(rewards.numel() == n && dones.numel() == n && truncated.numel() == n &&
                  events.numel() == n,
              "sparrow: per-copy outputs must hold N entries");
  auto stream = c10::cuda::getCurrentCUDAStream(dev.index());
  const int rc_ = g_api.env_step((SpEnv*)handle, actions.data_ptr<int64_t>(), states.data_ptr<float>(),
                          store_states.data_ptr<float>(), rewards.data_ptr<double>(),
                          (uint8_t*)dones.data_ptr(), (uint8_t*)truncated.data_ptr(),
                          (int8_t*)events.data_ptr(), (void*)stream.stream());
  check_rc(rc_, "env_step");
}

void rb_append(int64_t handle, const at::Tensor& s, const at::Tensor& a, const at::Tensor& r,
               const at::Tensor& s2, const at::Tensor& d) {
  TORCH_CHECK(g_api.rb_append, "sparrow: call sparrow::bind first");
  const at::Device dev = s.device();
  TORCH_CHECK(dev.is_cuda(), "sparrow: transitions must be CUDA tensors");
  const int64_t n = s.size(0);
  need(s, at::kFloat, "states", dev);
  need(s2, at::kFloat, "next_states", dev);
  need(a, at::kLong, "actions", dev);
  need(d, at::kBool, "dones", dev);
  TORCH_CHECK(r.device() == dev && r.is_contiguous() &&
                  (r.scalar_type() == at::kFloat || r.scalar_type() == at::kDouble),
              "sparrow: rewards must be contiguous float32/float64 on ", dev);
  TORCH_CHECK(a.numel() == n && r.numel() == n && s2.size(0) == n && d.numel() == n,
              "transition fields have mismatched lengths");  // replay.py:55-58
  auto stream = c10::cuda::getCurrentCUDAStream(dev.index());
  check_rc(g_api.rb_append((SpReplay*)handle, s.data_ptr<float>(), a.data_ptr<int64_t>(),
                           r.data_ptr(), r.scalar_type() == at::kDouble ? 1 : 0,
                           s2.data_ptr<float>(), (const uint8_t*)d.data_ptr(), n,
                           (void*)stream.stream()),
           "rb_append");
}

}  // namespace

void env_step_cpu(int64_t, const at::Tensor&, at::Tensor, at::Tensor, at::Tensor, at::Tensor,
                  at::Tensor, at::Tensor) {
  TORCH_CHECK(false, "sparrow: env_step needs CUDA tensors (there is no CPU path)");
}
void rb_append_cpu(int64_t, const at::Tensor&, const at::Tensor&, const at::Tensor&,
                   const at::Tensor&, const at::Tensor&) {
  TORCH_CHECK(false, "sparrow: rb_append needs CUDA tensors (there is no CPU path)");
}

TORCH_LIBRARY(sparrow, m) {
  m.def("bind(str lib_path) -> ()", &bind);
  m.def(
      "env_step(int handle, Tensor actions, Tensor(a!) states, Tensor(b!) store_states, "
      "Tensor(c!) rewards, Tensor(d!) dones, Tensor(e!) truncated, Tensor(f!) events) -> ()");
  m.def("rb_append(int handle, Tensor s, Tensor a, Tensor r, Tensor s2, Tensor d) -> ()");
}

// Kernels per dispatch key.  Autograd falls through: these ops write
// simulator outputs, nothing differentiable.  As for every PyTorch op, the
// (a!) .. (f!) outputs must be distinct tensors: torch crashes unwinding an
// error raised by an op whose mutable arguments alias, so VecEnv rejects
// states == store_states before the call (the C-ABI itself returns SP_EINVAL).
TORCH_LIBRARY_IMPL(sparrow, CUDA, m) {
  m.impl("env_step", &env_step);
  m.impl("rb_append", &rb_append);
}
TORCH_LIBRARY_IMPL(sparrow, CPU, m) {
  m.impl("env_step", &env_step_cpu);
  m.impl("rb_append", &rb_append_cpu);
}
TORCH_LIBRARY_IMPL(sparrow, Autograd, m) {
  m.impl("env_step", torch::CppFunction::makeFallthrough());
  m.impl("rb_append", torch::CppFunction::makeFallthrough());
}
