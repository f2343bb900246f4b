// Run I/O around the GPU path: PRSPAR01 arrays,
// headerless CSV, the training driver with the reference's run directory
// (free_energy.csv, checkpoint cadence, final arrays, prsp-manifest-1) and
// run reloading for inference. Host C++; the EM steps run on the engines.
//
// Reference: array_io.cpp:53-176 (arrays, CSV, format_double, trace),
// run_io.cpp:47-230 (manifest, DirectoryLogger, load_run, train_run),
// em.cpp:27-77 (the EM loop), annealing.cpp (schedules), model.cpp:77-232
// (parameter arrays, weight noise), sha256.cpp (data hash).
#pragma once
#include <cstdint>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace bscgpu {

struct Array {
  uint64_t rows = 0, cols = 0;
  std::vector<double> data;  // row-major
};

void save_array(const std::string& path, const double* data, uint64_t rows, uint64_t cols);
Array load_array(const std::string& path);
Array load_csv(const std::string& path);
Array load_dataset(const std::string& path);  // PRSPAR01 by magic, else CSV
std::string format_double(double v);          // shortest round-trip (std::to_chars)
std::string sha256_hex(const void* data, size_t n);
std::string sha256_hex_file(const std::string& path);

// Piecewise-linear schedule over the fraction of the budget (annealing.cpp:22-52).
struct Schedule {
  std::vector<std::pair<double, double>> anchors;
  void validate() const;
  double value_at(double position) const;
};

struct RunConfig {
  std::string model = "bsc";
  uint32_t dim = 0, latents = 0, hprime = 0, gamma = 0;
  std::vector<double> values;  // dsc alphabet
  uint64_t iterations = 0, seed = 0;
  uint32_t workers = 1, shards = 1;
  std::optional<double> tolerance;
  Schedule temperature{{{0.0, 1.0}}};
  Schedule w_noise{{{0.0, 0.0}}};
  double soft_winner_rho = 0.0;  // mca
  int device = 0;
  std::string data_file, data_sha256;
  uint64_t data_rows = 0, data_cols = 0;
};

struct NamedArray {
  std::string name;
  Array a;
};

struct TrainResult {
  std::vector<double> trace, seconds;
  std::vector<NamedArray> params;  // params_to_arrays order
};

void write_manifest(const std::string& path, const RunConfig& cfg, const std::vector<std::string>& files);
RunConfig read_manifest(const std::string& path);

// train_run (run_io.cpp:196-230) with the model's steps on the GPU engine.
TrainResult train_run(RunConfig& cfg, const double* y, uint64_t n, uint64_t d, const std::string& data_file,
                      const std::string& out_dir);

struct TrainedRun {
  RunConfig config;
  std::vector<NamedArray> params;
};
TrainedRun load_run(const std::string& dir);
// prsp_infer (capi.cpp:389-407): MAP states and masses of a trained run on new data.
void infer_run(const TrainedRun& run, const double* y, uint64_t n, uint64_t d, double* map_states, double* map_mass,
               double* expected, int device);

}  // namespace bscgpu
