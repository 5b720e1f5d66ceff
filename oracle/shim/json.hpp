// TEST INFRASTRUCTURE ONLY (oracle build shim).
// The reference includes `<json.hpp>` from its git-ignored `vendor/` directory
// (`/root/reference/proj/CMakeLists.txt:10`, `.gitignore:2`), which is absent.
// nlohmann/json ships in this image inside the cudnn_frontend wheel; the oracle
// Makefile adds that directory to the include path and this forwards to it.
#pragma once
#include <nlohmann/json.hpp>
