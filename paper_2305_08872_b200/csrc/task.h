// task.h — the task-text recogniser shared by task.cpp and the C-ABI.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amlt_gpu.h"

namespace amltk {

struct TaskError : std::runtime_error {
    amlt_status code;
    TaskError(amlt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct RecognizedTask {
    amlt_body_desc desc{};
    std::string a, b, r, thres, dis;  // array names per role ("" when absent)
    // AMLT_BODY_GENERIC: the statement term as a CUDA expression over
    // `a`, `b` and the aux leaves `c.v[q]` (one IEEE operation per syntax
    // tree node, in the tree's order), and the aux leaves in first-use order.
    std::string expr;
    std::vector<std::string> aux_names;
    std::vector<int> aux_class;  // amlt_leaf_class
    // the reference's compiled program for the statement: instructions per
    // opcode (AMLT_PROG_*), their total, and its body-op flops
    int prog_counts[AMLT_PROG_NOPS] = {};
    int prog_instrs = 0;
    int prog_flops = 0;
};

// Parse + recognise; throws TaskError (UNSUPPORTED / ENGINE).
RecognizedTask recognize_task(const std::string& source);

}  // namespace amltk
