// TEST INFRASTRUCTURE ONLY: the reference includes <json.hpp> from its
// un-vendored vendor/ directory (proj/.gitignore:2); this forwards to the
// nlohmann json single header that is on disk in this image (a third-party
// copy shipped inside cudnn_frontend; the include path is set by ref_build.sh).
#pragma once
#include <nlohmann/json.hpp>
