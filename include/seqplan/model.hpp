// seqplan/model.hpp — transformer shape vocabulary of the ISP block.
//
// Drop-in restatement of proj/include/seqplan/model.hpp (the reference's L0
// domain model): same names, same validation messages, same exception type.
// Added for the executor: the SwiGLU block tensor table used to shard weights.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace seqplan {

/// Model and batch shape (reference: model.hpp:12-48).
struct ModelConfig {
    std::int64_t hidden_dim = 0;           // H
    std::int64_t layers = 0;               // L
    std::int64_t heads = 0;                // D
    std::int64_t vocab = 0;                // V
    std::int64_t seq_len = 0;              // S (tokens)
    std::int64_t global_batch_tokens = 0;  // B (tokens)
    std::int64_t bytes_per_element = 2;    // e

    std::vector<std::string> validation_errors() const {
        std::vector<std::string> out;
        const std::pair<std::int64_t, const char*> fields[] = {
            {hidden_dim, "hidden_dim"}, {layers, "layers"},   {heads, "heads"},
            {vocab, "vocab"},           {seq_len, "seq_len"}, {global_batch_tokens, "global_batch_tokens"},
            {bytes_per_element, "bytes_per_element"}};
        for (const auto& [value, name] : fields)
            if (value <= 0) out.emplace_back(std::string(name) + " must be strictly positive");
        const bool both_positive = hidden_dim > 0 && heads > 0;
        if (both_positive && hidden_dim % heads != 0)
            out.emplace_back("hidden_dim must be divisible by heads");
        return out;
    }

    bool valid() const { return validation_errors().empty(); }

    void ensure_valid() const {
        const auto errors = validation_errors();
        if (errors.empty()) return;
        std::string text = "invalid model config:";
        for (const auto& e : errors) text += " " + e + ";";
        throw std::invalid_argument(text);
    }
};

/// Parameters of one layer as the reference counts them: QKV 3H^2, output H^2,
/// ratio-4 MLP 8H^2, two norms 2H (reference: model.hpp:58-63).
inline std::int64_t layer_param_count(const ModelConfig& cfg) {
    const std::int64_t h = cfg.hidden_dim;
    return h * (12 * h + 2);
}

/// Layers plus embedding and head (reference: model.hpp:66-68).
inline std::int64_t total_param_count(const ModelConfig& cfg) {
    return cfg.layers * layer_param_count(cfg) + 2 * cfg.hidden_dim * cfg.vocab;
}

// ---------------------------------------------------------------------------
// ISP block tensor table (executor addition).
// ---------------------------------------------------------------------------

/// The seven weight tensors of the LLaMA/InternLM block the executor runs:
/// RMSNorm weights, fused QKV, output projection, SwiGLU gate/up/down.
enum class BlockTensor : int { Norm1 = 0, Qkv, Out, Norm2, Gate, Up, Down };
constexpr int kBlockTensorCount = 7;

struct TensorShape {
    std::int64_t rows = 0;
    std::int64_t cols = 0;
    std::int64_t numel() const { return rows * cols; }
};

/// Row-major shape of each block tensor for hidden H and MLP width I.
inline std::array<TensorShape, kBlockTensorCount> block_tensor_shapes(std::int64_t H,
                                                                       std::int64_t I) {
    return {TensorShape{1, H}, TensorShape{3 * H, H}, TensorShape{H, H}, TensorShape{1, H},
            TensorShape{I, H}, TensorShape{I, H},     TensorShape{H, I}};
}

/// Psi_blk = 4H^2 + 3HI + 2H (SwiGLU block; SURVEY.md §8 preamble).
inline std::int64_t block_param_count(std::int64_t H, std::int64_t I) {
    return 4 * H * H + 3 * H * I + 2 * H;
}

}  // namespace seqplan
