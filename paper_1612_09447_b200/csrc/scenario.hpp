#pragma once

#include <string>
#include <utility>
#include <vector>

#include "gpu_system.hpp"

namespace eqsb {

// proj/include/eqs/metrics.hpp:13-28
struct StepMetrics {
  long step = 0;
  double t = 0, dt = 0;
  std::string method;
  bool accepted = false;
  int stages = 0, newton_iters = 0;
  long m_solves = 0, pcg_iters = 0;
  double rho = 0;
  std::string estimator_mode;
  int estimator_rank = 0;
  double err_est = 0;
  double t_residual = 0, t_solve = 0, t_setup = 0, t_estimator = 0;
};

// proj/include/eqs/scenario.hpp:67-81
struct RunResult {
  int exit_code = 0;
  std::string error;
  long accepted = 0, rejected = 0, stages = 0;
  SolveStats stats;
  std::vector<StepMetrics> steps;
  std::vector<SolveRecord> solves;
  std::vector<std::pair<double, std::vector<double>>> probe_rows;
  std::vector<double> final_x_free;
  double final_t = 0, wall_time = 0;
};

RunResult run_scenario(const SimConfig& config, const std::string& out_dir, int device);
const char* estimator_mode_name(int m);

}  // namespace eqsb
