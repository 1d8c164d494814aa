// TEST INFRASTRUCTURE (drop-in proof, not product code): the reference's own command-line run
// (config.hpp parse_config + runner.hpp run_case, unmodified except for the one-line patch that
// oracle/Makefile applies to a build-time copy of runner.hpp: the Stepper in run_case becomes
// ibm_b200::Stepper). Everything around the stepper — config parsing, the run loop, forces.csv,
// vorticity snapshots, checkpoints — is the reference's code; every step runs on the B200 path.
//   run_case_b200 <case.cfg> <out_dir> <n_steps>
#include <cstdio>
#include <cstdlib>

#include "ibm/runner.hpp"  // the patched copy (oracle/_ref/patched/ibm/runner.hpp)

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s case.cfg out_dir n_steps\n", argv[0]);
        return 2;
    }
    ibm::CaseConfig cfg = ibm::parse_config(argv[1]);
    ibm::RunOptions opts;
    opts.out_dir_override = argv[2];
    opts.n_steps_override = std::atoi(argv[3]);
    opts.quiet = true;
    const ibm::RunResult r = ibm::run_case(cfg, opts);
    std::printf("run_case_b200: exit %d, steps %d, solve-2 iterations %ld, last cd %.10f\n", r.exit_code,
                r.steps_done, (long)r.total_solve2_iters, r.last_cd);
    return r.exit_code;
}
