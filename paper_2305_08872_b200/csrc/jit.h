// jit.h — run-time compiled bodies for recognised statements that are not one
// of the fixed bodies (AMLT_BODY_GENERIC).
#pragma once

#include <string>
#include <vector>

#include "task.h"
#include "variants.h"

namespace amltk {

struct JitBody {
    std::string key;
    int dtype = 0;
    bool has_at = false;          // aux leaves indexed by i or (i, j): per-output state
    std::vector<int> variants;    // registry indices
    const BodyAux* aux = nullptr; // assign / naive kernels, reduce / pack shared per dtype
    bool loaded = false;          // kernel handles resolved (needs a device)
    double compile_seconds = 0;
    std::vector<char> cubin;      // NVRTC output, kept for a later load
    std::vector<std::string> lowered;
};

// Generates, compiles (NVRTC, sm_100a) and registers the kernels of a
// generated body; cached per (statement term, aux classes, dtype). With
// load == false (dry-run contexts) it compiles and registers but leaves the
// kernel handles unresolved. Throws TaskError(UNSUPPORTED / ENGINE / CUDA).
const JitBody& jit_body(const RecognizedTask& rt, int dtype, bool load);

// The CUDA source jit_body compiles for a statement (for inspection/tests).
std::string jit_source(const RecognizedTask& rt, int dtype);

}  // namespace amltk
