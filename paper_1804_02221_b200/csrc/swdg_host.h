// swdg_host.h — host helpers shared by the context and the structured mesh path.
#pragma once

#include <vector>

#include "../../include/swdg_gpu.h"

namespace swdg_host {
std::vector<swdg_face> structured_faces(int kx, int ky, bool px, bool py);
}
