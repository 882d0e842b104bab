// rollout/errors.hpp — drop-in error convention of the reference
// (proj/include/rollout/errors.hpp:10-59): every domain error derives from
// rollout::Error and carries a stable machine-readable code(). This header
// declares the codes the trainer-side scoring path raises or forwards, plus
// the four it adds (cuda_error, nccl_error, shape_mismatch, peer_failed).
#pragma once

#include <stdexcept>
#include <string>
#include <utility>

namespace rollout {

class Error : public std::runtime_error {
 public:
  Error(std::string code, const std::string& message) : std::runtime_error(message), code_(std::move(code)) {}
  const std::string& code() const noexcept { return code_; }

 private:
  std::string code_;
};

namespace detail {
template <const char* Code>
struct CodedError : Error {
  explicit CodedError(const std::string& message = Code) : Error(Code, message) {}
};
inline constexpr char kMalformedTurn[] = "malformed_turn";
inline constexpr char kMalformedRequest[] = "malformed_request";
inline constexpr char kIncompleteGroup[] = "incomplete_group";
inline constexpr char kCudaError[] = "cuda_error";
inline constexpr char kNcclError[] = "nccl_error";
inline constexpr char kShapeMismatch[] = "shape_mismatch";
inline constexpr char kPeerFailed[] = "peer_failed";
}  // namespace detail

// Reference codes used on this path (errors.hpp:208, 232, 237 in the reference).
struct MalformedTurn : detail::CodedError<detail::kMalformedTurn> { using CodedError::CodedError; };
struct MalformedRequest : detail::CodedError<detail::kMalformedRequest> { using CodedError::CodedError; };
struct IncompleteGroup : detail::CodedError<detail::kIncompleteGroup> { using CodedError::CodedError; };
// New on the device path.
struct CudaError : detail::CodedError<detail::kCudaError> { using CodedError::CodedError; };
struct NcclError : detail::CodedError<detail::kNcclError> { using CodedError::CodedError; };
struct ShapeMismatch : detail::CodedError<detail::kShapeMismatch> { using CodedError::CodedError; };
// Another rank's step failed; this rank's all-reduced result is void.
struct PeerFailed : detail::CodedError<detail::kPeerFailed> { using CodedError::CodedError; };

}  // namespace rollout
